// scan_kernel.cuh -- the sm_100a PFAC match kernels: the one-pass scan and
// the candidate-walking pass of the two-pass pipeline (filter_kernel.cuh has
// the filter passes).
//
// Reference semantics: scan.cpp:20-51 (walk), :69-119 (scan), trie.hpp:68-79
// (transition).  One logical walk per text offset, as in the paper
// (PAPER.md:87-95).
//
// pfac_scan_kernel<GROUPED, IDENT, KW, PAIR, CANDS>: one cooperative,
// persistent launch with one CTA per SM.
//
// CANDS = false (one-pass).  Block-wide state is read-only: the start filter
// and the byte->symbol map in shared memory.  Everything else is per warp:
//   phase 1, per warp, over statically interleaved 8 KiB warp-tiles
//   (8 groups of 1 KiB; each lane owns two 16-start slices per group):
//     - lane 0 keeps kStages groups in flight with cp.async.bulk (TMA bulk
//       copies, mbarrier-tracked) into the warp's ring in shared memory;
//     - each lane reads its two slices (conflict-free 16-byte loads; the
//       overhang from the next lane by SHFL) and probes the start filter:
//       single probe per start, or pair probes (one per two starts) plus the
//       in-lane second role test;
//     - survivors are compacted in start order into a per-warp queue and
//       walked 32 at a time (Walker::flush): depth-k jump table, one node
//       record per text byte, bucket verification at the depth limit;
//     - a warp scan of the per-lane record counts appends the records, in
//       order, to the warp's private staging region in HBM; per tile the
//       record count and staging offset go to a small table.
// CANDS = true (walking pass): phase 1 takes units of kSuper tiles from an
//   atomic counter, loads their candidates (left by the filter pass), drops
//   those whose 4-byte prefix misses a shared-memory bitmap, and walks the
//   rest with the same Walker.
// Both: grid sync -> phase 2: per-CTA sums of the tile counts.
//   grid sync -> phase 3: each CTA scans its contiguous range of tiles and
//     copies their staged records to their final offsets, so the output is
//     in (start, length, id) order without a sort (the reference merges per
//     unit vectors and std::sorts, scan.cpp:104-111).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "hepfac.h"
#include "layout.hpp"

namespace hfb::gpu {

namespace cg = cooperative_groups;

#ifndef HFB_WARPS
#define HFB_WARPS 16
#endif
#ifndef HFB_STAGES
#define HFB_STAGES 2
#endif
constexpr uint32_t kWarps = HFB_WARPS; // warps per CTA (one CTA per SM)
constexpr uint32_t kThreads = kWarps * 32;
#ifndef HFB_CWARPS
#define HFB_CWARPS 32
#endif
constexpr uint32_t kCWarps = HFB_CWARPS; // warps per CTA of the candidate-walking pass (CANDS)
constexpr uint32_t kSliceStarts = 16;                // consecutive starts of one lane slice
constexpr uint32_t kSlices = 2;                       // slices per lane per group
constexpr uint32_t kLaneStarts = kSliceStarts * kSlices;
constexpr uint32_t kGroup = 32 * kLaneStarts;         // 1024 starts per warp group
constexpr uint32_t kSliceSpan = 32 * kSliceStarts;    // slice s of lane L = group bytes [s*512 + 16L, +16)
constexpr uint32_t kGroupsPerTile = 8;
constexpr uint32_t kTile = kGroup * kGroupsPerTile;   // 8192 starts per warp-tile
constexpr uint32_t kSuper = 8;                        // CANDS walk unit: 8 tiles (u16 offsets still fit)
#ifndef HFB_QUEUE
#define HFB_QUEUE 1024
#endif
constexpr uint32_t kQueue = HFB_QUEUE;                // per-warp candidate queue (tile offsets), >= kGroup
constexpr uint32_t kStages = HFB_STAGES;              // per-warp TMA ring depth (groups in flight)
constexpr uint32_t kStageBytes = kGroup + 16;         // a group + the key overhang, 16-aligned
constexpr uint32_t kRegRecords = 2;                   // records a lane keeps per walk round

struct ScanArgs {
    TrieView trie;
    const uint8_t* text; // 16-byte aligned, readable up to round_up(n_avail, 16) + 16
    uint64_t n_own;      // starts [0, n_own) are reported
    uint64_t n_avail;    // walks stop here (global text end or shard halo end)
    uint64_t g0;         // global offset of text[0]
    hepfac_match_t* out;
    uint64_t out_cap;
    hepfac_match_t* stage;  // gridDim.x * kWarps regions of warp_cap records
    uint64_t warp_cap;
    uint64_t n_tiles;
    uint32_t* tile_count;
    uint32_t* tile_slot;    // offset of the tile's records inside its warp's region
    unsigned long long* chunk_sum;
    unsigned long long* total;
    const unsigned long long* base_in; // records placed by earlier launches of a streamed scan
    unsigned long long* base_out;      // base_in + this launch's total (distinct word)
    unsigned long long* warp_need;     // max records any warp needed (overflow sizing)
    unsigned int* err;
    // CANDS launches: per-tile start candidates from pfac_pair_filter_kernel
    const uint16_t* cand;       // cand_warps regions of cand_cap tile-relative offsets
    const uint32_t* cand_key;   // their first 4 text bytes
    uint64_t cand_cap;
    const uint32_t* tile_ccount;
    const uint32_t* tile_cslot;
    uint32_t cand_warps;        // tile t's candidates live in region t % cand_warps
    uint64_t n_ftiles;          // filter tiles; n_tiles then counts walk units of kSuper tiles
    unsigned long long* unit_next; // dynamic unit counter (zero at launch)
    uint32_t* tile_region;      // staging region (warp) of each unit
    const uint32_t* packed;     // symbol-key mode: the text packed by pfac_pack_symbols_kernel, or null
                                // (direct-index mode: by pfac_pack_dna_kernel)
    const uint32_t* valid;      // direct-index mode: one bit per text byte, 1 = inside the alphabet
};

// ---- text and dictionary helpers --------------------------------------------------

// 4 text bytes at any offset (little-endian), from two aligned word loads.
// The text buffer is padded, so reading up to 7 bytes past n_avail is safe.
__device__ __forceinline__ uint32_t text_word(const ScanArgs& a, uint64_t pos)
{
    const uint32_t* p = reinterpret_cast<const uint32_t*>(a.text + (pos & ~3ull));
    const uint32_t sh = uint32_t(pos & 3u) * 8u;
    const uint32_t lo = __ldg(p);
    return sh ? __funnelshift_r(lo, __ldg(p + 1), sh) : lo;
}

__device__ __forceinline__ uint32_t tail_mask(uint32_t left) { return left >= 4 ? 0xFFFFFFFFu : (1u << (8 * left)) - 1u; }
// The aligned words holding text[start, start + 8), and that window from them.
__device__ __forceinline__ uint3 raw_window(const ScanArgs& a, uint64_t start)
{
    const uint32_t* p = reinterpret_cast<const uint32_t*>(a.text + (start & ~3ull));
    return make_uint3(__ldg(p), __ldg(p + 1), __ldg(p + 2));
}
__device__ __forceinline__ uint64_t window_of(uint3 w, uint64_t start)
{
    const uint32_t sh = uint32_t(start & 3u) * 8u;
    const uint32_t lo = sh ? __funnelshift_r(w.x, w.y, sh) : w.x, hi = sh ? __funnelshift_r(w.y, w.z, sh) : w.y;
    return (uint64_t(hi) << 32) | lo;
}

// The low min(max(left, 0), 4) bytes of a word.
__device__ __forceinline__ uint32_t byte_mask(int32_t left)
{
    return __funnelshift_lc(0xFFFFFFFFu, 0u, uint32_t(max(left, 0)) * 8u);
}

// text[start, start + len) == pattern id, 4 bytes per step (patterns are
// stored 4-byte aligned and zero padded in the image).
__device__ __noinline__ bool same_bytes(const ScanArgs& a, uint64_t start, uint32_t id, uint32_t len)
{
    const uint32_t* p = reinterpret_cast<const uint32_t*>(a.trie.pat_bytes + __ldg(a.trie.pat_off + id));
    for (uint32_t i = 0; i < len; i += 4)
        if ((text_word(a, start + i) ^ __ldg(p + i / 4)) & tail_mask(len - i)) return false;
    return true;
}

__device__ __forceinline__ bool same_at(const ScanArgs& a, uint64_t start, uint64_t off, uint32_t len);

// Shared terminal: identify the slice by its key, then confirm it (the
// reference's dictionary lookup, trie.hpp:103-107; a miss is its logic_error
// "terminal node spells no dictionary pattern", scan.cpp:34).
// PAR (the walking pass, where stage-2 matches resolve often): every load of
// a stage is issued before its first use -- the slice's words 32 bytes at a
// time, a probe's id and key together, the pattern's length and offset
// together.  The one-pass kernel keeps the compact sequential form (measured:
// the parallel one costs its register allocation 11% at c2).
template <bool PAR>
__device__ __noinline__ uint32_t resolve_slice(const ScanArgs& a, uint64_t start, uint32_t len)
{
    const TrieView& t = a.trie;
    uint64_t h = 0;
    if (PAR) {
        const uint32_t sh = uint32_t(start & 3u) * 8u;
        for (uint32_t i = 0; i < len; i += 32) {
            const uint32_t* tw = reinterpret_cast<const uint32_t*>(a.text + ((start + i) & ~3ull));
            const uint32_t nw = min(8u, (len - i + 3) / 4);
            uint32_t tx[9];
#pragma unroll
            for (uint32_t k = 0; k < 9; ++k) tx[k] = k <= nw ? __ldg(tw + k) : 0u; // padded text
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k)
                if (k < nw) {
                    const uint32_t w = sh ? __funnelshift_r(tx[k], tx[k + 1], sh) : tx[k];
                    h = slice_step(h, t.hmul, w & tail_mask(len - i - 4 * k));
                }
        }
    } else {
        for (uint32_t i = 0; i < len; i += 4) h = slice_step(h, t.hmul, text_word(a, start + i) & tail_mask(len - i));
    }
    const uint64_t key = slice_key(h, len);
    for (uint64_t s = mix64(key) & t.ht_mask;; s = (s + 1) & t.ht_mask) {
        const uint32_t id = __ldg(t.ht_id + s);
        if (PAR) {
            const uint64_t k2 = __ldg(t.ht_key + s);
            if (id == kNoId) return kNoId;
            if (k2 == key) {
                const uint32_t plen = __ldg(t.pat_len + id);
                const uint64_t poff = __ldg(t.pat_off + id);
                return (plen == len && same_at(a, start, poff, len)) ? id : kNoId;
            }
        } else {
            if (id == kNoId) return kNoId;
            if (__ldg(t.ht_key + s) == key)
                return (__ldg(t.pat_len + id) == len && same_bytes(a, start, id, len)) ? id : kNoId;
        }
    }
}

// Records of one walk round.  Every record of a walk has the walk's start,
// so the first kRegRecords keep only (length, id) in registers (Sink); a
// re-walk emits the rest straight to the staging region (WriteSink).  Two
// types, so the walk carries only the state its mode needs.
// (Keeping these records in shared-memory slots instead, to lower register
// pressure, measured 2-15% slower: c3, c4 sigma=4, c5 100k.)
struct Sink {
    uint32_t n = 0;
    uint32_t l0 = 0, i0 = 0, l1 = 0, i1 = 0;

    __device__ __forceinline__ void put(uint64_t, uint32_t l, uint32_t i)
    {
        if (n == 0) l0 = l, i0 = i;
        else if (n == 1) l1 = l, i1 = i;
        ++n;
    }
};
struct WriteSink {
    hepfac_match_t* dst;
    uint64_t at, cap;
    uint32_t skip;

    __device__ __forceinline__ void put(uint64_t s, uint32_t l, uint32_t i)
    {
        if (skip) {
            --skip;
            return;
        }
        if (at < cap) reinterpret_cast<uint4*>(dst)[at] = make_uint4(uint32_t(s), uint32_t(s >> 32), l, i);
        ++at;
    }
};

// text[start, start + len) == the pattern stored at byte offset `off`.
// 32 bytes per block with every load of the block issued before the first
// compare (one memory latency per block instead of one per word).
__device__ __forceinline__ bool same_at(const ScanArgs& a, uint64_t start, uint64_t off, uint32_t len)
{
    const uint32_t* p = reinterpret_cast<const uint32_t*>(a.trie.pat_bytes + off);
    const uint32_t sh = uint32_t(start & 3u) * 8u;
    for (uint32_t i = 0; i < len; i += 32) {
        const uint32_t* tw = reinterpret_cast<const uint32_t*>(a.text + ((start + i) & ~3ull));
        const uint32_t nw = min(8u, (len - i + 3) / 4); // pattern words in this block
        uint32_t t[9], pw[8];
#pragma unroll
        for (uint32_t k = 0; k < 9; ++k) t[k] = k <= nw ? __ldg(tw + k) : 0u; // padded text: safe to overread
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k) pw[k] = k < nw ? __ldg(p + i / 4 + k) : 0u;
        uint32_t diff = 0;
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k)
            if (k < nw) diff |= ((sh ? __funnelshift_r(t[k], t[k + 1], sh) : t[k]) ^ pw[k]) & tail_mask(len - i - 4 * k);
        if (diff) return false;
    }
    return true;
}

// Depth-limit verification (scan.cpp:37-49): bucket entries are pre-sorted by
// (length, id), which is the order the records must appear in.  One load
// gives the bucket's span, one load per entry its id, length and bytes.
template <class S>
__device__ __forceinline__ void verify_span(const ScanArgs& a, uint2 span, uint64_t start, S& sink)
{
    const TrieView& t = a.trie;
    // Every bucket pattern spells the node's depth-limit path (the walk just
    // matched it), so the compare starts at the last 4-byte boundary before
    // the limit (pattern bytes are stored 4-byte aligned).
    const uint32_t skip = t.depth_limit & ~3u;
    for (uint32_t k = span.x, e = span.x + span.y; k < e; ++k) {
        const uint4 en = __ldg(reinterpret_cast<const uint4*>(t.bk_entry) + k);
        if (start + en.y > a.n_avail) continue; // overhangs the text end (scan.cpp:43)
        if (same_at(a, start + skip, ((uint64_t(en.w) << 32) | en.z) + skip, en.y - skip))
            sink.put(a.g0 + start, en.y, en.x);
    }
}

template <class S>
__device__ __forceinline__ void verify_bucket(const ScanArgs& a, uint32_t node, uint64_t start, S& sink)
{
    const TrieView& t = a.trie;
    verify_span(a, __ldg(reinterpret_cast<const uint2*>(t.bk_span) + __ldg(t.bucket_of + node)), start, sink);
}

// One failure-less walk (scan.cpp:20-51).  Each step issues a single record
// load that yields both the current node's flags (terminal / bucket) and the
// transition for the next byte.  Text bytes come from a register window of 8
// (`win`, the caller's copy of text[start, start + 8)), refilled 8 bytes at a
// time, so a step waits on one load, not two.
//
// A walk may begin below the root: (node, depth) from the jump table, which
// is only used for depth <= min_emit, where nothing above can report.
template <bool GROUPED, bool IDENT, bool PAR, class S>
__device__ __forceinline__ void walk(const ScanArgs& a, const uint16_t* s_sym, uint64_t start, uint64_t win,
                                     uint32_t node, uint32_t depth, S& sink, uint32_t pend = kNoId)
{
    const TrieView& t = a.trie;
    const uint32_t room = uint32_t(min(a.n_avail - start, uint64_t(0x7FFFFFFF)));
    const uint32_t limit = t.depth_limit ? t.depth_limit : 0xFFFFFFFFu;
    uint32_t wpos = depth; // `win` holds text[start, start + 8)
    if (depth > 8) {       // symbol-key jumps start deeper: the window of the current byte
        win = (uint64_t(text_word(a, start + (depth & ~7u) + 4)) << 32) | text_word(a, start + (depth & ~7u));
        wpos = depth & 7u;
    }
    for (;;) {
        const bool more = depth < room;
        if (wpos == 8) { // next 8 bytes (the padded buffer makes the overread safe)
            win = (uint64_t(text_word(a, start + depth + 4)) << 32) | text_word(a, start + depth);
            wpos = 0;
        }
        const uint32_t byte = more ? uint32_t(win >> (8 * wpos)) & 0xFFu : 0u;
        const uint32_t sym = IDENT ? byte : uint32_t(s_sym[byte]);
        const bool step = more && (IDENT || sym != kNoSym);
        uint32_t word, base, meta, inline_id = kNoId;
        // the node's path id rides along with its record (same latency), so
        // keyed terminals rarely need the slice lookup
        const uint32_t pid = __ldg(t.path_id + node);
        if (GROUPED) {
            const uint32_t g = step ? (sym >> 6) : 0u;
            const uint4 r = __ldg(reinterpret_cast<const uint4*>(t.nodes) + (node * t.groups + g));
            const bool hi = (sym >> 5) & 1u;
            word = hi ? r.y : r.x;
            base = (r.z & kBaseMask) + (hi ? uint32_t(__popc(r.x)) : 0u);
            meta = r.z;
            inline_id = r.w;
        } else {
            const uint2 r = __ldg(reinterpret_cast<const uint2*>(t.nodes) + node);
            word = r.x;
            base = r.y & kBaseMask;
            meta = r.y;
        }
        if (pid != kKeep) pend = pid;
        if (depth && (meta & kFlagTerminal)) {
            uint32_t id = GROUPED ? inline_id : __ldg(t.term_id + node);
            if (id == kNoId) id = pend != kNoId ? pend : resolve_slice<PAR>(a, start, depth);
            if (id == kNoId) atomicOr(a.err, 1u);
            else sink.put(a.g0 + start, depth, id);
        }
        if (depth == limit) { // depth-limit nodes are leaves (scan.cpp:37-49)
            if (meta & kFlagBucket) verify_bucket(a, node, start, sink);
            break;
        }
        if (!step) break;
        const uint32_t b = sym & 31u;
        if (!((word >> b) & 1u)) break;
        node = base + uint32_t(__popc(word & ((1u << b) - 1u)));
        ++depth;
        ++wpos;
    }
}

// ---- start filter ------------------------------------------------------------

// Bit j set = start j of the lane slice may report.  w[0..5] = the slice's
// 16 bytes plus the next 8.  KW: 1 = k < 4, 2 = k in 5..8, 3 = k == 4.
template <int KW>
__device__ __forceinline__ uint32_t filter_mask(const TrieView& t, const uint32_t (&w)[6], const uint32_t* s_filter,
                                                uint32_t valid)
{
    if (KW == 0) return valid;
    const uint32_t k = t.filter_k;
    const uint32_t mask4 = (t.filter_words - 1u) << 2; // hash -> byte offset of the bitmap word
    const uint32_t m32 = (KW == 3 || k >= 4) ? 0xFFFFFFFFu : ((1u << (8 * k)) - 1u);
    const uint32_t mhi = k >= 8 ? 0xFFFFFFFFu : (k > 4 ? ((1u << (8 * (k - 4))) - 1u) : 0u);
    const uint8_t* fbytes = reinterpret_cast<const uint8_t*>(s_filter);
    uint32_t m[2] = {0u, 0u}; // start j ends up at bit 7 - j % 8 of m[j / 8]
#pragma unroll
    for (int j = 0; j < int(kSliceStarts); ++j) {
        const uint32_t lo = (j & 3) ? __funnelshift_r(w[j >> 2], w[(j >> 2) + 1], 8 * (j & 3)) : w[j >> 2];
        uint32_t key;
        if (KW == 2) {
            const uint32_t hi =
                ((j & 3) ? __funnelshift_r(w[(j >> 2) + 1], w[(j >> 2) + 2], 8 * (j & 3)) : w[(j >> 2) + 1]) & mhi;
            key = lo + hi * 0x85EBCA77u; // filter_fold (one IMAD)
        } else {
            key = KW == 3 ? lo : (lo & m32);
        }
        const uint32_t off = __umulhi(key, kFilterMul) & mask4; // filter_word(key) * 4
        const uint32_t word = *reinterpret_cast<const uint32_t*>(fbytes + off);
        m[j >> 3] = __funnelshift_l(__funnelshift_l(0u, word, key), m[j >> 3], 1); // MSB-first
    }
    return (__brev((m[0] << 24) | (m[1] << 16))) & valid; // start j at bit j
}

// 32-bit word at byte offset `off` of dynamic shared memory (the start
// filter table lives at offset 0).
__device__ __forceinline__ uint32_t table_word(uint32_t off)
{
    uint32_t v;
    asm("{\n\t.reg .u32 b;\n\tmov.u32 b, _ZN3hfb3gpu4smemE;\n\tadd.u32 b, b, %1;\n\tld.shared.u32 %0, [b];\n\t}"
        : "=r"(v)
        : "r"(off));
    return v;
}

// Pair form (layout.hpp): 8 probes for a 16-start slice.  Probe p reads the
// word of the middle at odd position i = 2p + 1 and tests start i - 1 (role A:
// bit of its first byte) and start i (role B: bit of its 4th byte).
// filter_pair returns bit j = start j passed its first role.
__device__ __forceinline__ uint32_t pair_offset(const TrieView& t, uint32_t mid)
{
    return ((mid * kPairMul) >> t.pair_shift) << 2; // pair_word(mid) * 4
}

__device__ __forceinline__ uint32_t filter_pair(const TrieView& t, const uint32_t (&w)[5], uint32_t valid)
{
    // Only the low 24 bits of a middle and the low 5 of an amount matter.
    auto window = [&](int n) -> uint32_t {
        switch (n & 3) {
        case 0: return w[n >> 2];
        case 1: return w[n >> 2] >> 8;
        case 2: return w[n >> 2] >> 16;
        default: return __funnelshift_r(w[n >> 2], w[(n >> 2) + 1], 24);
        }
    };
    uint32_t m0 = 0, m1 = 0; // two independent accumulator chains, MSB-first
#pragma unroll
    for (int i = 1; i < int(kSliceStarts); i += 2) {
        const uint32_t mid = window(i);
        const uint32_t amt_a = window(i - 1), amt_b = window(i + 3);
        const uint32_t word = table_word(pair_offset(t, mid));
        uint32_t& acc = i < 8 ? m0 : m1;
        acc = __funnelshift_l(__funnelshift_l(0u, word, amt_a), acc, 1); // start i - 1
        acc = __funnelshift_l(__funnelshift_l(0u, word, amt_b), acc, 1); // start i
    }
    return __brev((m0 << 24) | (m1 << 16)) & valid; // start j at bit j
}

// Second pair level: each survivor j of `mask` tests its other role (odd j:
// role A at the middle j + 1; even j: role B at the middle j), reading its 4
// bytes back from the staged lane slice `src` in shared memory.  Two
// survivors (the lowest and the highest) per round for latency overlap.
__device__ __forceinline__ bool pair_second_test(const TrieView& t, const uint8_t* src, uint32_t j)
{
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(src + (j & ~3u));
    const uint32_t y = __funnelshift_r(wp[0], wp[1], 8 * j); // bytes j..j+3 (shift wraps mod 32)
    const bool odd = j & 1u;
    const uint32_t mid = odd ? (y >> 8) : y;
    const uint32_t amt = odd ? y : (y >> 24);
    const uint32_t word = table_word(pair_offset(t, mid));
    return int32_t(word << (amt & 31u)) < 0;
}

__device__ __forceinline__ uint32_t filter_pair_second(const TrieView& t, uint32_t mask, const uint8_t* src)
{
    uint32_t keep = mask;
    for (uint32_t c = mask; c;) { // the lowest and the highest survivor per round
        const uint32_t lo = __ffs(c) - 1, hi = 31 - __clz(c);
        c &= ~((1u << lo) | (1u << hi));
        const bool ok_lo = pair_second_test(t, src, lo);
        const bool ok_hi = pair_second_test(t, src, hi);
        if (!ok_lo) keep &= ~(1u << lo);
        if (!ok_hi) keep &= ~(1u << hi);
    }
    return keep;
}

// ---- warp helpers ---------------------------------------------------------------

__device__ __forceinline__ uint32_t warp_exclusive(uint32_t v, uint32_t lane, uint32_t& total)
{
    uint32_t incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= uint32_t(d)) incl += u;
    }
    total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    return incl - v;
}

template <uint32_t NW>
__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* s_scr, uint32_t& total)
{
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t wt;
    const uint32_t ex = warp_exclusive(v, lane, wt);
    if (lane == 0) s_scr[warp] = wt;
    __syncthreads();
    if (warp == 0) {
        const uint32_t x = lane < NW ? s_scr[lane] : 0u;
        uint32_t tt;
        const uint32_t xe = warp_exclusive(x, lane, tt);
        if (lane < NW) s_scr[lane] = xe;
        if (lane == 0) s_scr[NW] = tt;
    }
    __syncthreads();
    total = s_scr[NW];
    const uint32_t r = s_scr[warp] + ex;
    __syncthreads();
    return r;
}

// ---- the walk stage of one warp ---------------------------------------------------

// Second-level filter probe of the start at global offset `start` (text read
// back from L2, where the TMA copy just streamed it).
template <int KW>
__device__ __forceinline__ bool probe2(const ScanArgs& a, uint64_t start)
{
    const TrieView& t = a.trie;
    const uint32_t k = t.filter_k;
    uint32_t key = text_word(a, start);
    if (KW == 1) key &= (1u << (8 * k)) - 1u;
    if (KW == 2) {
        const uint32_t mhi = k >= 8 ? 0xFFFFFFFFu : ((1u << (8 * (k - 4))) - 1u);
        key += (text_word(a, start + 4) & mhi) * 0x85EBCA77u; // filter_fold
    }
    const uint32_t slot = filter2_slot(key, t.filter2_bits);
    return (__ldg(t.filter2 + (slot >> 5)) >> (slot & 31u)) & 1u;
}

// The jump-table slot of the node a start reaches after its first k bytes
// (`win` = text[start, start + 8)); w.z == kNoId when no trie path spells them.
struct JumpHit {
    uint4 w;   // {lo, hi, node, term}
    uint4 aux; // {bk_first, bk_count, flags, pend}
    uint32_t slot;
};
// Cuckoo lookup (layout.hpp): both candidate slots load at once.  (Loading
// both slots' extensions here as well cost the fused kernel 40% on c2:
// register spills; emit_at_limit loads the chosen one.)
__device__ __forceinline__ JumpHit jump_lookup_key(const TrieView& t, uint32_t lo, uint32_t hi)
{
    const uint4* slots = reinterpret_cast<const uint4*>(t.jump);
    const uint32_t k32 = lo ^ (hi * 0x85EBCA77u);
    const uint32_t s1 = jump_slot(k32, t.jump_bits), s2 = jump_slot2(k32, t.jump_bits);
    JumpHit a, b;
    a.w = __ldg(slots + 2 * s1);
    a.aux = __ldg(slots + 2 * s1 + 1);
    a.slot = s1;
    b.w = __ldg(slots + 2 * s2);
    b.aux = __ldg(slots + 2 * s2 + 1);
    b.slot = s2;
    if (a.w.z != kNoId && a.w.x == lo && a.w.y == hi) return a;
    if (b.w.z != kNoId && b.w.x == lo && b.w.y == hi) return b;
    a.w.z = kNoId;
    return a;
}

// Symbol-key mode: the first filter_k symbols of the start, packed sym_bits
// each (the host's key, image.cpp).  False when one of those bytes is outside
// the alphabet: no trie path spells it (the packed filter input aliased it to
// symbol 0, so this is where such starts are dropped).
__device__ __forceinline__ bool symbol_key(const ScanArgs& a, const uint16_t* s_sym, uint64_t start, uint32_t& key)
{
    const TrieView& t = a.trie;
    const uint32_t k = t.filter_k, sb = t.sym_bits;
    bool ok = true;
    key = 0;
    for (uint32_t i = 0; i < k; i += 4) {
        const uint32_t w = text_word(a, start + i);
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b)
            if (i + b < k) {
                const uint32_t s = s_sym[(w >> (8 * b)) & 0xFFu];
                ok = ok && s != kNoSym;
                key |= (s == kNoSym ? 0u : s) << (sb * (i + b));
            }
    }
    return ok;
}

// Symbol-key mode: the start's key read from the packed text (packed word j
// holds the symbols of bytes [j * 32 / sym_bits, ...), LSB first).
__device__ __forceinline__ uint32_t packed_key(const ScanArgs& a, uint64_t start)
{
    const uint32_t sb = a.trie.sym_bits, kb = sb * a.trie.filter_k;
    const uint64_t bit = start * sb;
    const uint32_t* w = a.packed + (bit >> 5);
    const uint32_t v = __funnelshift_r(__ldg(w), __ldg(w + 1), uint32_t(bit & 31u));
    return kb >= 32 ? v : v & ((1u << kb) - 1u);
}

template <int KW>
__device__ __forceinline__ JumpHit jump_lookup(const TrieView& t, uint64_t win)
{
    const uint32_t k = t.filter_k;
    uint32_t lo = uint32_t(win), hi = 0;
    if (KW == 1) lo &= (1u << (8 * k)) - 1u;
    if (KW == 2) hi = uint32_t(win >> 32) & (k >= 8 ? 0xFFFFFFFFu : ((1u << (8 * (k - 4))) - 1u));
    return jump_lookup_key(t, lo, hi);
}

// A walk that starts at the depth limit (k == limit): the node's terminal
// record and its bucket come from the jump slot (walk() semantics at the
// limit: terminal first, then the bucket in (length, id) order).
template <bool PAR, class S>
__device__ __forceinline__ void emit_at_limit(const ScanArgs& a, const JumpHit& h, uint64_t start, uint32_t depth,
                                              S& sink)
{
    if (h.aux.z & 1u) {
        uint32_t id = h.w.w;
        if (id == kNoId) id = h.aux.w != kNoId ? h.aux.w : resolve_slice<PAR>(a, start, depth);
        if (id == kNoId) atomicOr(a.err, 1u);
        else sink.put(a.g0 + start, depth, id);
    }
    if (h.aux.z & 2u) verify_span(a, make_uint2(h.aux.x, h.aux.y), start, sink);
}

// A slot with an inline pattern list (flags bit 2, layout.hpp): the start's
// records are exactly the listed patterns that match the text, in list order.
// Their first 24 bytes from inline_skip came with the extension; the text words are
// L1 hits next to the window just read.  Pattern bytes are read only past
// those 24.
template <class S>
__device__ __forceinline__ void emit_inline(const ScanArgs& a, uint32_t slot, uint32_t flags, uint64_t start, S& sink)
{
    const TrieView& t = a.trie;
    const uint32_t skip = inline_skip(t.filter_k, t.sym_bits);
    const uint4* ext = reinterpret_cast<const uint4*>(t.jump_ext) + 4 * slot;
    const uint32_t cnt = (flags >> kJumpInlineShift) & 3u;
    uint4 x[4];
    x[0] = __ldg(ext);
    x[1] = __ldg(ext + 1);
    x[2] = cnt > 1 ? __ldg(ext + 2) : make_uint4(0u, 0u, 0u, 0u);
    x[3] = cnt > 1 ? __ldg(ext + 3) : make_uint4(0u, 0u, 0u, 0u);
    const uint64_t p = start + skip;
    const uint32_t* tw = reinterpret_cast<const uint32_t*>(a.text + (p & ~3ull));
    const uint32_t sh = uint32_t(p & 3u) * 8u;
    uint32_t raw[7], txt[6];
#pragma unroll
    for (uint32_t k = 0; k < 7; ++k) raw[k] = __ldg(tw + k); // padded text: safe to overread
#pragma unroll
    for (uint32_t k = 0; k < 6; ++k) txt[k] = sh ? __funnelshift_r(raw[k], raw[k + 1], sh) : raw[k];
#pragma unroll
    for (uint32_t j = 0; j < kJumpExtEntries; ++j) {
        if (j >= cnt) break;
        const uint4 e0 = x[2 * j], e1 = x[2 * j + 1];
        const uint32_t id = e0.x, len = e0.y;
        if (start + len > a.n_avail) continue; // overhangs the text end (scan.cpp:26, :43)
        const uint32_t pw[6] = {e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
        const int32_t rem = int32_t(len - skip);
        uint32_t diff = 0;
#pragma unroll
        for (uint32_t k = 0; k < 6; ++k) diff |= (txt[k] ^ pw[k]) & byte_mask(rem - int32_t(4 * k));
        if (!diff && (rem <= int32_t(kJumpExtBytes) ||
                      same_at(a, p + kJumpExtBytes, __ldg(t.pat_off + id) + skip + kJumpExtBytes,
                              uint32_t(rem) - kJumpExtBytes)))
            sink.put(a.g0 + start, len, id);
    }
}

// The walking pass (32 warps, 64 registers) keeps the inline check out of
// line: few of its candidates reach a slot, and inlined it spilled.  The
// sink goes in and comes back by value, so the caller's sink stays in
// registers (by reference it had to live in local memory for the whole walk).
template <class S>
__device__ __noinline__ S emit_inline_call(const ScanArgs& a, uint32_t slot, uint32_t flags, uint64_t start, S sink)
{
    emit_inline(a, slot, flags, start, sink);
    return sink;
}

template <bool PAR, class S>
__device__ __forceinline__ void emit_listed(const ScanArgs& a, const JumpHit& h, uint64_t start, S& sink)
{
#ifndef HFB_INLINE_ALL
    if (PAR) {
        sink = emit_inline_call(a, h.slot, h.aux.z, start, sink);
        return;
    }
#endif
    emit_inline(a, h.slot, h.aux.z, start, sink);
}

template <bool GROUPED, bool IDENT, int KW, bool PAR, class S>
__device__ __forceinline__ void run_start(const ScanArgs& a, const uint16_t* s_sym, uint64_t start, uint64_t win,
                                          S& sink);

// A start with more records than the registers hold (rare): run it again
// from its offset and write records kRegRecords.. directly.  Out of line, so
// each flush carries one copy of the walk, and nothing of the first run
// (jump slot, node, window) has to stay live for it.
template <bool GROUPED, bool IDENT, int KW, bool PAR>
__device__ __noinline__ void rewalk_rest(const ScanArgs& a, const uint16_t* s_sym, uint64_t start,
                                         hepfac_match_t* region, uint64_t at)
{
    WriteSink wr{region, at, a.warp_cap, kRegRecords};
    run_start<GROUPED, IDENT, KW, PAR>(a, s_sym, start, window_of(raw_window(a, start), start), wr);
}

// Every record of one start (`win` = text[start, start + 8)): the depth-k
// jump (byte keys, or packed symbol keys), then the slot's inline list, the
// depth-limit emit, or a walk from the jump node (from the root without a
// jump table).
template <bool GROUPED, bool IDENT, int KW, bool PAR, class S>
__device__ __forceinline__ void run_start(const ScanArgs& a, const uint16_t* s_sym, uint64_t start, uint64_t win,
                                          S& sink)
{
    uint32_t node = 0, depth = 0;
    JumpHit hit{};
    hit.aux.w = kNoId; // no jump: the walk starts at the root with no path id
    if (KW != 0 && a.trie.jump_bits) {
        // (grouped records mean sigma > 32: never symbol keys)
        if (!GROUPED && a.trie.sym_bits && a.packed) {
            // the key from the packed text (2 loads, not k symbol lookups);
            // bytes outside the alphabet were packed as symbol 0, so a hit is
            // checked byte by byte -- by the inline compare itself, or here
            hit = jump_lookup_key(a.trie, packed_key(a, start), 0u);
            uint32_t key;
            if (hit.w.z != kNoId && !(hit.aux.z & kJumpInline) && !symbol_key(a, s_sym, start, key)) hit.w.z = kNoId;
        } else if (!GROUPED && a.trie.sym_bits) {
            uint32_t key;
            if (symbol_key(a, s_sym, start, key)) hit = jump_lookup_key(a.trie, key, 0u);
            else hit.w.z = kNoId;
        } else {
            hit = jump_lookup<KW>(a.trie, win);
        }
        node = hit.w.z;
        depth = a.trie.filter_k;
    }
    if (node == kNoId) return;
    // k == limit: walks end at the jump node; the slot has what they emit
    const bool at_limit = KW != 0 && a.trie.jump_bits && a.trie.filter_k == a.trie.depth_limit;
    if (hit.aux.z & kJumpInline) emit_listed<PAR>(a, hit, start, sink);
    else if (at_limit) emit_at_limit<PAR>(a, hit, start, depth, sink);
    else walk<GROUPED, IDENT, PAR>(a, s_sym, start, win, node, depth, sink, hit.aux.w);
}

template <bool GROUPED, bool IDENT, int KW, bool PAR>
struct Walker {
    const ScanArgs& a;
    const uint16_t* s_sym;
    uint16_t* q; // this warp's candidate queue: start offsets inside the current tile
    uint32_t lane;
    hepfac_match_t* region;
    uint64_t cursor; // records this warp has staged so far

    // Candidates [0, n) of the tile starting at `lo`: second-level probe,
    // then walk the survivors and append their records in start order.
    __device__ __forceinline__ void flush(uint64_t lo, uint32_t n)
    {
        uint32_t ns = n;
        if (KW != 0 && a.trie.filter2_bits) {
            ns = 0;
            const uint32_t below = (1u << lane) - 1u;
            for (uint32_t r0 = 0; r0 < n; r0 += 32) {
                const uint32_t e = r0 + lane;
                uint16_t off = 0;
                bool keep = false;
                if (e < n) {
                    off = q[e];
                    keep = probe2<KW>(a, lo + off);
                }
                const uint32_t b = __ballot_sync(0xFFFFFFFFu, keep);
                __syncwarp(); // every read of this round is done (and ordered) before the in-place writes
                if (keep) q[ns + __popc(b & below)] = off;          // compaction in place, order kept
                ns += __popc(b);
            }
            __syncwarp();
        }
        // The fused kernel loads each round's text windows one round ahead,
        // so a candidate's jump lookup does not wait for its text (c2 +2.5%;
        // the walking pass, at 64 registers, lost 1-3% with it).
        uint3 pre = make_uint3(0u, 0u, 0u);
        if (!PAR && lane < ns) pre = raw_window(a, lo + q[lane]);
        for (uint32_t r0 = 0; r0 < ns; r0 += 32) {
            const uint32_t e = r0 + lane;
            uint3 cur = pre;
            if (!PAR && e + 32 < ns) pre = raw_window(a, lo + q[e + 32]);
            if (PAR && e < ns) cur = raw_window(a, lo + q[e]);
            Sink sink;
            uint64_t start = 0;
            if (e < ns) {
                start = lo + q[e];
                run_start<GROUPED, IDENT, KW, PAR>(a, s_sym, start, window_of(cur, start), sink);
            }
            uint32_t tot;
            const uint32_t ex = warp_exclusive(sink.n, lane, tot);
            if (sink.n) {
                const uint64_t at = cursor + ex;
                const uint64_t g = a.g0 + start;
                uint4* dst = reinterpret_cast<uint4*>(region);
                if (at < a.warp_cap) dst[at] = make_uint4(uint32_t(g), uint32_t(g >> 32), sink.l0, sink.i0);
                if (sink.n > 1 && at + 1 < a.warp_cap)
                    dst[at + 1] = make_uint4(uint32_t(g), uint32_t(g >> 32), sink.l1, sink.i1);
                if (sink.n > kRegRecords) // rare: run the start again and write the rest directly
                    rewalk_rest<GROUPED, IDENT, KW, PAR>(a, s_sym, start, region, at + kRegRecords);
            }
            cursor += tot;
        }
        __syncwarp();
    }
};

// Phases 2 and 3 of every cooperative scan kernel (after phase 1 staged each
// tile's records in its warp's region and wrote tile_count / tile_slot):
//   grid sync -> phase 2: per-CTA sums of the tile counts over contiguous
//     ranges of tiles;
//   grid sync -> phase 3: each CTA scans its range and copies the staged
//     records to their final offsets, so the output is in (start, length,
//     id) order without a sort (the reference merges per-unit vectors and
//     std::sorts, scan.cpp:104-111).
// Tile i was staged by warp tile_region[i] (CANDS: dynamic units) or by
// warp i % (grid * NW) (static interleave).
template <uint32_t NW, bool CANDS>
__device__ __forceinline__ void place_records(const ScanArgs& a, uint32_t* s_scr)
{
    constexpr uint32_t NT = NW * 32;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    // phase 2: per-CTA sums over contiguous chunks of tiles
    cg::grid_group grid = cg::this_grid();
    grid.sync();
    const uint64_t nt = a.n_tiles, chunk = (nt + gridDim.x - 1) / gridDim.x;
    const uint64_t c0 = min(nt, uint64_t(blockIdx.x) * chunk), c1 = min(nt, c0 + chunk);
    {
        uint32_t s = 0;
        for (uint64_t i = c0 + tid; i < c1; i += NT) s += a.tile_count[i];
        uint32_t tot;
        block_exclusive<NW>(s, s_scr, tot);
        if (tid == 0) a.chunk_sum[blockIdx.x] = tot;
    }
    grid.sync();

    // phase 3: scan the chunk, copy staged slices to their final offsets
    // warp 0 sums the CTA sums (before this CTA, and all) for the whole CTA
    __shared__ unsigned long long s_base[2];
    if (warp == 0) {
        unsigned long long before = 0, all = 0;
        for (uint32_t b = lane; b < gridDim.x; b += 32) {
            const unsigned long long v = a.chunk_sum[b];
            before += b < blockIdx.x ? v : 0ull;
            all += v;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            before += __shfl_xor_sync(0xFFFFFFFFu, before, d);
            all += __shfl_xor_sync(0xFFFFFFFFu, all, d);
        }
        if (lane == 0) s_base[0] = before, s_base[1] = all;
    }
    __syncthreads();
    const unsigned long long origin = *a.base_in;
    unsigned long long base = origin + s_base[0];
    const unsigned long long total = s_base[1];
    if (blockIdx.x == gridDim.x - 1 && tid == 0) {
        *a.total = total;
        *a.base_out = origin + total;
    }
    const bool fits = origin + total <= a.out_cap && *a.warp_need == 0;
    for (uint64_t r0 = c0; r0 < c1; r0 += NT) {
        const uint64_t i = r0 + tid;
        const uint32_t n = i < c1 ? a.tile_count[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive<NW>(n, s_scr, tot);
        if (n && fits) {
            const uint64_t region = CANDS ? a.tile_region[i] : i % (uint64_t(gridDim.x) * NW);
            const uint4* src = reinterpret_cast<const uint4*>(a.stage + region * a.warp_cap) + a.tile_slot[i];
            uint4* dst = reinterpret_cast<uint4*>(a.out) + base + ex;
#pragma unroll 4
            for (uint32_t k = 0; k < n; ++k) dst[k] = src[k];
        }
        base += tot;
    }
}

// ---- PTX helpers: per-warp TMA bulk ring --------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    // The stage's previous contents were consumed before the warp's
    // __syncwarp, so the copy cannot overwrite data still being read.
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Shared-memory bytes a CTA needs beyond the filter bitmap.
constexpr uint32_t smem_fixed_bytes(bool cands)
{
    return cands ? kCWarps * kQueue * 2 + 512 : kWarps * kStages * kStageBytes + kWarps * kQueue * 2 + 512;
}

// CANDS = false: the fused scan (filter, walks, ordered output) over text.
// CANDS = true: the second pass of the pair pipeline -- walks the candidates
// pfac_pair_filter_kernel left per tile; no filter, no text staging.
template <bool GROUPED, bool IDENT, int KW, bool PAIR, bool CANDS = false>
__global__ void __launch_bounds__(CANDS ? kCWarps * 32 : kThreads, 1) pfac_scan_kernel(const __grid_constant__ ScanArgs a)
{
    constexpr uint32_t NW = CANDS ? kCWarps : kWarps, NT = NW * 32;
    extern __shared__ __align__(128) uint8_t smem[];
    // first in shared memory: the start filter (fused) or the 4-byte-prefix bitmap (CANDS)
    const uint32_t fwords = CANDS ? a.trie.key4_words : (KW ? a.trie.filter_words : 0u);
    uint32_t* s_filter = reinterpret_cast<uint32_t*>(smem);                   // first: 2^bits / 8 bytes
    uint8_t* s_ring = smem + size_t(fwords) * 4;                               // [warp][stage][kStageBytes]
    uint16_t* s_queue = reinterpret_cast<uint16_t*>(s_ring + (CANDS ? 0u : NW * kStages * kStageBytes));
    uint16_t* s_sym = s_queue + NW * kQueue;                                   // [256]
    __shared__ uint64_t s_bar[CANDS ? 1 : NW][kStages];
    __shared__ uint32_t s_scr[NW + 1];

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const TrieView& t = a.trie;
    for (uint32_t i = tid; i < fwords; i += NT) s_filter[i] = __ldg((CANDS ? t.key4 : t.filter) + i);
    if (!IDENT)
        for (uint32_t i = tid; i < 256; i += NT) s_sym[i] = __ldg(t.symtab + i);

    const uint64_t me = t.min_emit;
    const uint64_t start_end = a.n_avail >= me ? min(a.n_own, a.n_avail - me + 1) : 0;
    const uint64_t avail16 = (a.n_avail + 15) & ~15ull;
    const uint32_t gw = blockIdx.x * NW + warp, W = gridDim.x * NW;
    uint8_t* ring = s_ring + warp * kStages * kStageBytes;
    uint64_t* bars = s_bar[CANDS ? 0 : warp];

    // Producer (lane 0): the warp's groups -- tiles gw, gw + W, ..., 8 groups
    // each, up to `stop` -- with kStages in flight.  The consumer below visits
    // exactly the same groups in the same order.
    const uint64_t stop = min(avail16, a.n_tiles * uint64_t(kTile));
    uint64_t p_addr = uint64_t(gw) * kTile;
    uint32_t p_g = 0, p_stage = 0;
    const uint64_t p_skip = uint64_t(W - 1) * kTile;
    auto produce = [&]() {
        if (p_addr >= stop) return;
        const uint32_t n = uint32_t(min(uint64_t(kStageBytes), avail16 - p_addr));
        bulk_load(ring + p_stage * kStageBytes, a.text + p_addr, n, &bars[p_stage]);
        p_stage = p_stage + 1 == kStages ? 0u : p_stage + 1;
        p_addr += kGroup;
        if (++p_g == kGroupsPerTile) p_g = 0, p_addr += p_skip;
    };
    if (lane == 0 && !CANDS) {
        for (uint32_t s = 0; s < kStages; ++s) mbar_init(&bars[s]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint32_t s = 0; s < kStages; ++s) produce();
    }
    __syncthreads(); // filter, symbol map and barrier inits visible

    Walker<GROUPED, IDENT, KW, CANDS> wk{a, s_sym, s_queue + warp * kQueue, lane, a.stage + uint64_t(gw) * a.warp_cap, 0};
    if constexpr (CANDS) {
        // Walk units of kSuper filter tiles: lane i < kSuper fetches tile i's
        // candidate count and slot, so one load latency covers the unit, and
        // rounds are filled across tile boundaries.
        // Units are handed out dynamically (warps finish unevenly: walks
        // are latency chains); the unit records which region staged it.
        for (;;) {
            uint64_t unit = 0;
            if (lane == 0) unit = atomicAdd(a.unit_next, 1ull);
            unit = __shfl_sync(0xFFFFFFFFu, unit, 0);
            if (unit >= a.n_tiles) break;
            const uint64_t lo = unit * uint64_t(kSuper) * kTile;
            const uint64_t slot = wk.cursor;
            const uint64_t ft = unit * kSuper + lane;
            uint32_t cnt = 0, cslot = 0;
            if (lane < kSuper && ft < a.n_ftiles) cnt = a.tile_ccount[ft], cslot = a.tile_cslot[ft];
            uint32_t pre = cnt; // inclusive prefix over lanes 0..kSuper-1
#pragma unroll
            for (uint32_t d = 1; d < kSuper; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, pre, d);
                if (lane >= d) pre += u;
            }
            uint32_t total = __shfl_sync(0xFFFFFFFFu, pre, kSuper - 1);
            pre -= cnt; // exclusive
            if (total <= kQueue) {
                // every entry of the unit loaded at once: entry f belongs to
                // the last tile i with pre_i <= f (lane i < kSuper holds
                // pre_i and tile i's slot; a 3-step search over shuffles)
                static_assert(kSuper == 8, "the tile search takes 3 steps");
                // Entries are re-checked against the 4-byte-prefix bitmap
                // (one shared-memory probe) and compacted in order: most
                // pair survivors are false positives, and each would cost
                // an L2 round trip in the walk.
                const uint32_t kmask4 = (fwords - 1u) << 2;
                const uint8_t* kbytes = reinterpret_cast<const uint8_t*>(s_filter);
                uint32_t kept = 0;
                for (uint32_t f0 = 0; f0 < total; f0 += 32) {
                    const uint32_t f = f0 + lane;
                    bool keep = false;
                    uint16_t v = 0;
                    uint32_t i = 0;
#pragma unroll
                    for (uint32_t step = kSuper / 2; step; step >>= 1)
                        if (f >= __shfl_sync(0xFFFFFFFFu, pre, i + step)) i += step;
                    const uint32_t p_i = __shfl_sync(0xFFFFFFFFu, pre, i), s_i = __shfl_sync(0xFFFFFFFFu, cslot, i);
                    if (f < total) {
                        const uint64_t t_i = unit * kSuper + i;
                        const uint64_t at = (t_i % a.cand_warps) * a.cand_cap + s_i + (f - p_i);
                        v = uint16_t(a.cand[at] + i * kTile);
                        keep = true;
                        if (fwords) {
                            // symbol keys are re-hashed: the filter pass
                            // already used this hash of the same key
                            uint32_t key = a.cand_key[at];
                            if (!GROUPED && a.trie.sym_bits) key = filter2_hash(key);
                            const uint32_t word =
                                *reinterpret_cast<const uint32_t*>(kbytes + (__umulhi(key, kFilterMul) & kmask4));
                            keep = int32_t(word << (key & 31u)) < 0;
                        }
                    }
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
                    if (keep) wk.q[kept + __popc(bal & ((1u << lane) - 1u))] = v;
                    kept += __popc(bal);
                }
                total = kept;
                if (total) {
                    __syncwarp();
                    wk.flush(lo, total);
                }
            } else {
                uint32_t qn = 0;
                for (uint32_t i = 0; i < kSuper; ++i) {
                    const uint32_t n_i = __shfl_sync(0xFFFFFFFFu, cnt, i);
                    if (n_i == 0) continue;
                    const uint32_t s_i = __shfl_sync(0xFFFFFFFFu, cslot, i);
                    const uint64_t t_i = unit * kSuper + i;
                    const uint16_t* src = a.cand + (t_i % a.cand_warps) * a.cand_cap + s_i;
                    for (uint32_t c0 = 0; c0 < n_i;) {
                        if (qn == kQueue) {
                            __syncwarp();
                            wk.flush(lo, qn);
                            qn = 0;
                        }
                        const uint32_t n = min(kQueue - qn, n_i - c0);
                        for (uint32_t k = lane; k < n; k += 32) wk.q[qn + k] = uint16_t(src[c0 + k] + i * kTile);
                        qn += n;
                        c0 += n;
                    }
                }
                if (qn) {
                    __syncwarp();
                    wk.flush(lo, qn);
                }
            }
            if (lane == 0) {
                a.tile_count[unit] = uint32_t(wk.cursor - slot);
                a.tile_slot[unit] = uint32_t(slot);
                a.tile_region[unit] = gw;
            }
        }
    }
    uint32_t c_stage = 0, c_parity = 0;
    for (uint64_t tile = gw; !CANDS && tile < a.n_tiles; tile += W) {
        const uint64_t lo = tile * kTile;
        const uint64_t slot = wk.cursor;
        // tile-relative limits (32-bit): starts that may report, groups fetched
        const uint32_t rem = start_end > lo ? uint32_t(min(start_end - lo, uint64_t(kTile))) : 0u;
        const uint32_t fetched = uint32_t(min((stop - lo + kGroup - 1) / kGroup, uint64_t(kGroupsPerTile)));
        uint32_t qn = 0;
        // g == fetched is the tile's last flush: one call site keeps one
        // inlined copy of the walk in the kernel
        for (uint32_t g = 0;; ++g) {
            if (g == fetched) {
                if (qn) wk.flush(lo, qn);
                break;
            }
            // slice s of this lane: group starts [s * 512 + 16 * lane, +16)
            uint32_t valid[kSlices];
#pragma unroll
            for (uint32_t sl = 0; sl < kSlices; ++sl) {
                const int32_t r = int32_t(rem) - int32_t(g * kGroup + sl * kSliceSpan + lane * kSliceStarts);
                valid[sl] = r >= int32_t(kSliceStarts) ? 0xFFFFu : (r > 0 ? (1u << r) - 1u : 0u);
            }
            mbar_wait(&bars[c_stage], c_parity);
            uint32_t mask[kSlices] = {};
            if (__any_sync(0xFFFFFFFFu, valid[0] | valid[kSlices - 1])) {
                // Conflict-free 16-byte reads (a quarter-warp covers 128
                // contiguous bytes); each slice's overhang comes from the next
                // lane, the last lane's from lane 0's next slice or the tail.
                const uint8_t* stage = ring + c_stage * kStageBytes;
                uint4 v[kSlices];
#pragma unroll
                for (uint32_t sl = 0; sl < kSlices; ++sl)
                    v[sl] = *reinterpret_cast<const uint4*>(stage + sl * kSliceSpan + lane * kSliceStarts);
                const uint2 tail = *reinterpret_cast<const uint2*>(stage + kGroup);
                const uint32_t nxt = (lane + 1) & 31u;
#pragma unroll
                for (uint32_t sl = 0; sl < kSlices; ++sl) {
                    const bool last = sl + 1 == kSlices;
                    const uint32_t sx = (lane == 0 && !last) ? v[sl + 1].x : v[sl].x;
                    const uint32_t sy = (lane == 0 && !last) ? v[sl + 1].y : v[sl].y;
                    uint32_t ox = __shfl_sync(0xFFFFFFFFu, sx, nxt);
                    uint32_t oy = __shfl_sync(0xFFFFFFFFu, sy, nxt);
                    if (last && lane == 31) ox = tail.x, oy = tail.y;
                    if (PAIR) {
                        const uint32_t w[5] = {v[sl].x, v[sl].y, v[sl].z, v[sl].w, ox};
                        mask[sl] = filter_pair(t, w, valid[sl]);
                    } else {
                        const uint32_t w[6] = {v[sl].x, v[sl].y, v[sl].z, v[sl].w, ox, oy};
                        mask[sl] = filter_mask<KW>(t, w, s_filter, valid[sl]);
                    }
                }
                if (PAIR) {
#pragma unroll
                    for (uint32_t sl = 0; sl < kSlices; ++sl)
                        mask[sl] = filter_pair_second(t, mask[sl], stage + sl * kSliceSpan + lane * kSliceStarts);
                }
            }
            __syncwarp();
            if (lane == 0) produce(); // the stage is consumed: refill it
            if (++c_stage == kStages) c_stage = 0, c_parity ^= 1u;
            static_assert(kSlices == 2, "survivor counts pack into two 16-bit fields");
            uint32_t packed = 0; // per-slice survivor counts, 16 bits each
#pragma unroll
            for (uint32_t sl = 0; sl < kSlices; ++sl) packed |= uint32_t(__popc(mask[sl])) << (16 * sl);
            if (__any_sync(0xFFFFFFFFu, packed)) { // queue the candidates, in start order (slice, lane, j)
                uint32_t tot_packed;
                const uint32_t ex = warp_exclusive(packed, lane, tot_packed);
                uint32_t tot = 0;
#pragma unroll
                for (uint32_t sl = 0; sl < kSlices; ++sl) tot += (tot_packed >> (16 * sl)) & 0xFFFFu;
                if (qn + tot > kQueue) { // warp-uniform
                    wk.flush(lo, qn);
                    qn = 0;
                }
                uint32_t base = qn;
#pragma unroll
                for (uint32_t sl = 0; sl < kSlices; ++sl) {
                    uint32_t at = base + ((ex >> (16 * sl)) & 0xFFFFu);
                    const uint32_t first = g * kGroup + sl * kSliceSpan + lane * kSliceStarts;
                    for (uint32_t m = mask[sl]; m; m &= m - 1) wk.q[at++] = uint16_t(first + __ffs(m) - 1);
                    base += (tot_packed >> (16 * sl)) & 0xFFFFu;
                }
                qn += tot;
                __syncwarp();
            }
        }
        if (lane == 0) {
            a.tile_count[tile] = uint32_t(wk.cursor - slot);
            a.tile_slot[tile] = uint32_t(slot);
        }
    }
    if (lane == 0 && wk.cursor > a.warp_cap) atomicMax(a.warp_need, (unsigned long long)wk.cursor);

    place_records<NW, CANDS>(a, s_scr);
}

// Evicts the text from L2 between timed iterations when it would fit there.
__global__ void l2_flush_kernel(uint4* buf, size_t n16, uint32_t salt)
{
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
        buf[i] = make_uint4(salt, uint32_t(i), 0u, 0u);
}

} // namespace hfb::gpu

// scan_kernel.cuh -- the sm_100a PFAC match kernel.
//
// Reference semantics: scan.cpp:20-51 (walk), :69-119 (scan), trie.hpp:68-79
// (transition).  One logical walk per text offset, as in the paper
// (PAPER.md:87-95); the GPU work decomposition:
//
//   persistent CTAs (256 threads) claim 4 KiB tiles of start offsets in order
//   from a global counter, so tile t is only claimed after tiles < t;
//   1. stage the tile + a 64-byte halo of text into shared memory;
//   2. each thread owns 16 consecutive starts and tests each against the
//      start filter (one shared-memory bit probe on the first k bytes);
//   3. survivors walk the trie image (one 8/16-byte __ldg per text byte,
//      L2-resident for configs 1-4) and COUNT their matches;
//   4. block scan of the counts, then a decoupled look-back over the
//      per-tile status words gives the tile's global output offset, so the
//      output is written directly in (start, length, id) order: no sort pass
//      (replaces the reference's merge + std::sort, scan.cpp:104-111);
//   5. threads with matches re-walk their survivors and write the records.
#pragma once

#include <cuda/atomic>
#include <cuda_runtime.h>

#include "hepfac.h"
#include "layout.hpp"

namespace hfb::gpu {

constexpr uint32_t kThreads = 256;
constexpr uint32_t kPerThread = 16;
constexpr uint32_t kTile = kThreads * kPerThread; // start offsets per tile
constexpr uint32_t kSmemHalo = 64;                // text bytes staged past the tile
constexpr uint32_t kSmemText = kTile + kSmemHalo;

// Tile status word: [epoch:16][flag:2][count:46].  The epoch tags the launch,
// so the array never needs clearing between launches.
constexpr unsigned long long kFlagAggregate = 1ull << 46;
constexpr unsigned long long kFlagPrefix = 2ull << 46;
constexpr unsigned long long kFlagMask = 3ull << 46;
constexpr unsigned long long kCountMask = (1ull << 46) - 1;
constexpr unsigned long long kEpochMask = ~((1ull << 48) - 1);

struct ScanArgs {
    TrieView trie;
    const uint8_t* text; // 16-byte aligned, readable up to round_up(n_avail, 16)
    uint64_t n_own;      // starts [0, n_own) are reported
    uint64_t n_avail;    // walks stop here (global text end or shard halo end)
    uint64_t g0;         // global offset of text[0]
    hepfac_match_t* out;
    uint64_t out_cap;
    unsigned long long* status;
    unsigned long long* tile_ctr;
    unsigned long long tile_base;
    unsigned long long n_tiles;
    unsigned long long epoch_bits;
    unsigned long long* total;
    unsigned int* err;
};

struct TileCtx {
    const uint8_t* s_text;
    const uint16_t* s_sym;
    uint64_t lo;
    uint32_t s_len;
};

__device__ __forceinline__ uint32_t text_byte(const ScanArgs& a, const TileCtx& c, uint64_t pos)
{
    const uint64_t r = pos - c.lo;
    return r < c.s_len ? uint32_t(c.s_text[r]) : uint32_t(__ldg(a.text + pos));
}

__device__ __forceinline__ void put_match(const ScanArgs& a, uint64_t at, uint64_t start, uint32_t len,
                                          uint32_t id)
{
    if (at >= a.out_cap) return; // overflow: host re-runs with the exact capacity
    uint4 v;
    v.x = uint32_t(start);
    v.y = uint32_t(start >> 32);
    v.z = len;
    v.w = id;
    reinterpret_cast<uint4*>(a.out)[at] = v;
}

__device__ __noinline__ bool same_bytes(const ScanArgs& a, const TileCtx& c, uint64_t start, uint32_t id,
                                        uint32_t len)
{
    const uint8_t* p = a.trie.pat_bytes + __ldg(a.trie.pat_off + id);
    for (uint32_t i = 0; i < len; ++i)
        if (text_byte(a, c, start + i) != uint32_t(__ldg(p + i))) return false;
    return true;
}

// Shared terminal: identify the slice by its key, then confirm byte-wise
// (the reference's dictionary lookup, trie.hpp:103-107; a miss is its
// logic_error "terminal node spells no dictionary pattern", scan.cpp:34).
__device__ __noinline__ uint32_t resolve_slice(const ScanArgs& a, const TileCtx& c, uint64_t start,
                                               uint32_t len, uint64_t h)
{
    const TrieView& t = a.trie;
    const uint64_t key = slice_key(h, len);
    for (uint64_t s = mix64(key) & t.ht_mask;; s = (s + 1) & t.ht_mask) {
        const uint32_t id = __ldg(t.ht_id + s);
        if (id == kNoId) return kNoId;
        if (__ldg(t.ht_key + s) == key)
            return (__ldg(t.pat_len + id) == len && same_bytes(a, c, start, id, len)) ? id : kNoId;
    }
}

// Depth-limit verification (scan.cpp:37-49): bucket ids are pre-sorted by
// (length, id), which is the order the records must appear in.
template <bool WRITE>
__device__ __noinline__ uint32_t verify_bucket(const ScanArgs& a, const TileCtx& c, uint32_t node,
                                               uint64_t start, uint64_t at)
{
    const TrieView& t = a.trie;
    const uint32_t b = __ldg(t.bucket_of + node);
    uint32_t found = 0;
    for (uint32_t k = __ldg(t.bk_start + b), e = __ldg(t.bk_start + b + 1); k < e; ++k) {
        const uint32_t id = __ldg(t.bk_ids + k);
        const uint32_t len = __ldg(t.pat_len + id);
        if (start + len > a.n_avail) continue; // overhangs the text end (scan.cpp:43)
        if (!same_bytes(a, c, start, id, len)) continue;
        if (WRITE) put_match(a, at + found, a.g0 + start, len, id);
        ++found;
    }
    return found;
}

// One failure-less walk (scan.cpp:20-51).  Each step issues a single record
// load that yields both the current node's flags (terminal / bucket) and the
// transition for the next byte.
template <bool GROUPED, bool IDENT, bool WRITE>
__device__ __forceinline__ uint32_t walk(const ScanArgs& a, const TileCtx& c, uint64_t start, uint64_t at)
{
    const TrieView& t = a.trie;
    uint32_t node = 0, depth = 0, found = 0;
    uint64_t pos = start, h = 0;
    for (;;) {
        const bool more = pos < a.n_avail;
        const uint32_t byte = more ? text_byte(a, c, pos) : 0u;
        const uint32_t sym = IDENT ? byte : uint32_t(c.s_sym[byte]);
        const bool step = more && (IDENT || sym != kNoSym);
        uint32_t word, base, meta, inline_id = kNoId;
        if (GROUPED) {
            const uint32_t g = step ? (sym >> 6) : 0u;
            const uint4 r = __ldg(reinterpret_cast<const uint4*>(t.nodes) + size_t(node) * t.groups + g);
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
        if (depth) {
            if (meta & kFlagTerminal) {
                uint32_t id = GROUPED ? inline_id : __ldg(t.term_id + node);
                if (id == kNoId) id = resolve_slice(a, c, start, depth, h);
                if (id == kNoId) {
                    atomicOr(a.err, 1u);
                } else {
                    if (WRITE) put_match(a, at + found, a.g0 + start, depth, id);
                    ++found;
                }
            }
            if (depth == t.depth_limit) {
                if (meta & kFlagBucket) found += verify_bucket<WRITE>(a, c, node, start, at + found);
                break;
            }
        }
        if (!step) break;
        const uint32_t b = sym & 31u;
        if (!((word >> b) & 1u)) break;
        node = base + uint32_t(__popc(word & ((1u << b) - 1u)));
        ++pos;
        ++depth;
        h = slice_step(h, t.hmul, byte);
    }
    return found;
}

// Start filter over a thread's 16 starts: bit j set = start j may report.
template <int KW>
__device__ __forceinline__ uint32_t filter_mask(const ScanArgs& a, const uint8_t* s_text,
                                                const uint32_t* s_filter, uint32_t base, uint32_t valid)
{
    if (KW == 0) return valid;
    const uint4 q = *reinterpret_cast<const uint4*>(s_text + base);
    const uint2 r = *reinterpret_cast<const uint2*>(s_text + base + 16);
    const uint32_t w[6] = {q.x, q.y, q.z, q.w, r.x, r.y};
    const uint32_t k = a.trie.filter_k, bits = a.trie.filter_bits;
    const uint32_t m32 = k >= 4 ? 0xFFFFFFFFu : ((1u << (8 * k)) - 1u);
    const uint64_t m64 = k >= 8 ? ~0ull : ((1ull << (8 * k)) - 1ull);
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < int(kPerThread); ++j) {
        const uint32_t lo = __funnelshift_r(w[j >> 2], w[(j >> 2) + 1], 8 * (j & 3));
        uint32_t slot;
        if (KW == 1) {
            slot = filter_slot32(lo & m32, bits);
        } else {
            const uint32_t hi = __funnelshift_r(w[(j >> 2) + 1], w[(j >> 2) + 2], 8 * (j & 3));
            slot = filter_slot64(((uint64_t(hi) << 32) | lo) & m64, bits);
        }
        m |= ((s_filter[slot >> 5] >> (slot & 31u)) & 1u) << j;
    }
    return m & valid;
}

// Decoupled look-back (single-pass ordered scan): publish this tile's
// aggregate, then fold predecessors 32 at a time until an inclusive prefix is
// found.  Executed by one full warp.
__device__ __forceinline__ uint64_t look_back(const ScanArgs& a, uint64_t tile, uint64_t agg, uint32_t lane)
{
    using ref = cuda::atomic_ref<unsigned long long, cuda::thread_scope_device>;
    if (tile == 0) {
        if (lane == 0) ref(a.status[0]).store(a.epoch_bits | kFlagPrefix | agg, cuda::memory_order_relaxed);
        return 0;
    }
    if (lane == 0) ref(a.status[tile]).store(a.epoch_bits | kFlagAggregate | agg, cuda::memory_order_relaxed);
    uint64_t excl = 0;
    long long top = (long long)tile - 1;
    for (;;) {
        const long long idx = top - (long long)lane;
        unsigned long long s = a.epoch_bits | kFlagPrefix; // virtual prefix 0 before tile 0
        if (idx >= 0) s = ref(a.status[idx]).load(cuda::memory_order_relaxed);
        const bool ready = (s & kEpochMask) == a.epoch_bits && (s & kFlagMask) != 0;
        if (__any_sync(0xFFFFFFFFu, !ready)) {
            __nanosleep(32);
            continue;
        }
        const uint32_t pre = __ballot_sync(0xFFFFFFFFu, (s & kFlagMask) == kFlagPrefix);
        uint64_t v = s & kCountMask;
        if (pre && lane > uint32_t(__ffs(pre) - 1)) v = 0;
#pragma unroll
        for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
        excl += v;
        if (pre) break;
        top -= 32;
    }
    if (lane == 0)
        ref(a.status[tile]).store(a.epoch_bits | kFlagPrefix | (excl + agg), cuda::memory_order_relaxed);
    return excl;
}

template <bool GROUPED, bool IDENT, int KW>
__global__ void __launch_bounds__(kThreads) pfac_scan_kernel(const __grid_constant__ ScanArgs a)
{
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t fwords = KW ? a.trie.filter_words : 0u;
    uint32_t* s_filter = reinterpret_cast<uint32_t*>(smem);
    uint16_t* s_sym = reinterpret_cast<uint16_t*>(smem + fwords * 4);
    uint8_t* s_text = smem + fwords * 4 + (IDENT ? 0u : 512u);
    __shared__ uint32_t s_warp[kThreads / 32];
    __shared__ unsigned long long s_base, s_tile;

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    for (uint32_t i = tid; i < fwords; i += kThreads) s_filter[i] = __ldg(a.trie.filter + i);
    if (!IDENT)
        for (uint32_t i = tid; i < 256; i += kThreads) s_sym[i] = __ldg(a.trie.symtab + i);

    // Starts that can still reach a reporting depth before the text ends.
    const uint64_t me = a.trie.min_emit;
    const uint64_t start_end = a.n_avail >= me ? min(a.n_own, a.n_avail - me + 1) : 0;

    for (;;) {
        if (tid == 0) s_tile = atomicAdd(a.tile_ctr, 1ull) - a.tile_base;
        __syncthreads();
        const unsigned long long tile = s_tile;
        if (tile >= a.n_tiles) break;
        const uint64_t lo = tile * kTile;
        const uint64_t avail16 = (a.n_avail + 15) & ~15ull;
        const uint32_t nbytes = uint32_t(min(uint64_t(kSmemText), avail16 - lo));
        const uint4* src = reinterpret_cast<const uint4*>(a.text + lo);
        for (uint32_t i = tid; i < nbytes / 16; i += kThreads) reinterpret_cast<uint4*>(s_text)[i] = __ldg(src + i);
        __syncthreads();
        const TileCtx c{s_text, s_sym, lo, nbytes};

        const uint64_t o0 = lo + uint64_t(tid) * kPerThread;
        uint32_t valid = 0;
        if (o0 < start_end) {
            const uint64_t r = start_end - o0;
            valid = r >= kPerThread ? 0xFFFFu : ((1u << r) - 1u);
        }
        const uint32_t mask = valid ? filter_mask<KW>(a, s_text, s_filter, tid * kPerThread, valid) : 0u;

        uint32_t cnt = 0;
        for (uint32_t m = mask; m; m &= m - 1)
            cnt += walk<GROUPED, IDENT, false>(a, c, o0 + uint32_t(__ffs(m) - 1), 0);

        // block exclusive scan of per-thread counts
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= uint32_t(d)) incl += v;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const uint32_t v = lane < kThreads / 32 ? s_warp[lane] : 0u;
            uint32_t vi = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, vi, d);
                if (lane >= uint32_t(d)) vi += u;
            }
            if (lane < kThreads / 32) s_warp[lane] = vi - v;
            const uint64_t agg = __shfl_sync(0xFFFFFFFFu, vi, kThreads / 32 - 1);
            const uint64_t excl = look_back(a, tile, agg, lane);
            if (lane == 0) {
                s_base = excl;
                if (tile == a.n_tiles - 1) *a.total = excl + agg;
            }
        }
        __syncthreads();
        if (cnt) {
            uint64_t at = s_base + s_warp[warp] + (incl - cnt);
            for (uint32_t m = mask; m; m &= m - 1)
                at += walk<GROUPED, IDENT, true>(a, c, o0 + uint32_t(__ffs(m) - 1), at);
        }
    }
}

// Evicts the text from L2 between timed iterations when it would fit there.
__global__ void l2_flush_kernel(uint4* buf, size_t n16, uint32_t salt)
{
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
        buf[i] = make_uint4(salt, uint32_t(i), 0u, 0u);
}

} // namespace hfb::gpu

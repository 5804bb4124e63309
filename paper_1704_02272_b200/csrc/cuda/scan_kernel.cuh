// scan_kernel.cuh -- the sm_100a PFAC match kernel.
//
// Reference semantics: scan.cpp:20-51 (walk), :69-119 (scan), trie.hpp:68-79
// (transition).  One logical walk per text offset, as in the paper
// (PAPER.md:87-95).  GPU work decomposition (one cooperative, persistent
// launch; 512-thread CTAs, 8 KiB tiles of start offsets):
//
//   phase 1, per tile (tiles claimed in order from a global counter; the next
//   claim and its text are always in flight while the current tile runs):
//     a. the tile's text + a 64-byte halo arrive in shared memory by
//        cp.async.bulk (TMA bulk copy) into a double buffer, mbarrier-tracked;
//     b. every thread owns 16 consecutive starts and probes the start filter
//        (bitmap in shared memory, 2 hashes of the first k bytes);
//     c. survivors are compacted block-wide, in start order, into a queue;
//     d. queue entries are split evenly over the threads and walked through
//        the GPU trie image (one 8/16-byte __ldg per text byte); each thread
//        keeps its first few records in registers;
//     e. a block scan of the per-thread counts orders the tile's records; one
//        atomicAdd reserves the tile's slice of a staging buffer.
//   grid sync -> phase 2: exclusive scan of the per-tile counts.
//   grid sync -> phase 3: each tile's staged slice is copied to its final
//     offset, so the output is in (start, length, id) order with no sort
//     (replaces the reference's merge + std::sort, scan.cpp:104-111) and no
//     tile ever waits on another tile inside phase 1.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "hepfac.h"
#include "layout.hpp"

namespace hfb::gpu {

namespace cg = cooperative_groups;

constexpr uint32_t kThreads = 512;
constexpr uint32_t kWarps = kThreads / 32;
constexpr uint32_t kPerThread = 16;
constexpr uint32_t kTile = kThreads * kPerThread; // start offsets per tile
constexpr uint32_t kSmemHalo = 64;                // text bytes staged past the tile
constexpr uint32_t kSmemText = kTile + kSmemHalo;
constexpr uint32_t kRegRecords = 2; // records a thread buffers before re-walking

struct ScanArgs {
    TrieView trie;
    const uint8_t* text; // 16-byte aligned, readable up to round_up(n_avail, 16)
    uint64_t n_own;      // starts [0, n_own) are reported
    uint64_t n_avail;    // walks stop here (global text end or shard halo end)
    uint64_t g0;         // global offset of text[0]
    hepfac_match_t* out;
    hepfac_match_t* stage;
    uint64_t cap; // records out / stage can hold
    unsigned long long* tile_ctr;
    unsigned long long tile_base;
    unsigned long long n_tiles;
    uint32_t* tile_count;
    unsigned long long* tile_slot;  // staging offset of each tile's records
    unsigned long long* tile_first; // final offset of each tile's records
    unsigned long long* chunk_sum;  // one per CTA
    unsigned long long* stage_cursor;
    unsigned long long* total;
    unsigned int* err;
};

// ---- small PTX helpers (TMA bulk copy + mbarrier) --------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
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

// ---- walk --------------------------------------------------------------------

struct TileCtx {
    const uint8_t* s_text;
    const uint16_t* s_sym;
    uint64_t lo;
    uint32_t s_len; // bytes of text valid in s_text (0 = read everything from global)
};

__device__ __forceinline__ uint32_t text_byte(const ScanArgs& a, const TileCtx& c, uint64_t pos)
{
    const uint64_t r = pos - c.lo;
    return r < c.s_len ? uint32_t(c.s_text[r]) : uint32_t(__ldg(a.text + pos));
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

// Record sink: the first kRegRecords records of a thread stay in registers;
// `skip` lets a re-walk drop the records that were already kept.
struct Sink {
    uint32_t n = 0;
    uint4 r0, r1; // the first kRegRecords (= 2) records, as stored
    // write mode (re-walk of an overflowing thread)
    hepfac_match_t* dst = nullptr;
    uint64_t at = 0, cap = 0;
    uint32_t skip = 0;

    __device__ __forceinline__ void put(uint64_t s, uint32_t l, uint32_t i)
    {
        const uint4 v = make_uint4(uint32_t(s), uint32_t(s >> 32), l, i);
        if (dst) {
            if (skip) {
                --skip;
            } else {
                if (at < cap) reinterpret_cast<uint4*>(dst)[at] = v;
                ++at;
            }
            return;
        }
        if (n == 0) r0 = v;
        else if (n == 1) r1 = v;
        ++n;
    }
};

// Depth-limit verification (scan.cpp:37-49): bucket ids are pre-sorted by
// (length, id), which is the order the records must appear in.
__device__ __forceinline__ void verify_bucket(const ScanArgs& a, const TileCtx& c, uint32_t node, uint64_t start,
                                              Sink& sink)
{
    const TrieView& t = a.trie;
    const uint32_t b = __ldg(t.bucket_of + node);
    for (uint32_t k = __ldg(t.bk_start + b), e = __ldg(t.bk_start + b + 1); k < e; ++k) {
        const uint32_t id = __ldg(t.bk_ids + k);
        const uint32_t len = __ldg(t.pat_len + id);
        if (start + len > a.n_avail) continue; // overhangs the text end (scan.cpp:43)
        if (same_bytes(a, c, start, id, len)) sink.put(a.g0 + start, len, id);
    }
}

// One failure-less walk (scan.cpp:20-51).  Each step issues a single record
// load that yields both the current node's flags (terminal / bucket) and the
// transition for the next byte.
template <bool GROUPED, bool IDENT>
__device__ __forceinline__ void walk(const ScanArgs& a, const TileCtx& c, uint64_t start, Sink& sink)
{
    const TrieView& t = a.trie;
    uint32_t node = 0, depth = 0;
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
                if (id == kNoId) atomicOr(a.err, 1u);
                else sink.put(a.g0 + start, depth, id);
            }
            if (depth == t.depth_limit) {
                if (meta & kFlagBucket) verify_bucket(a, c, node, start, sink);
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
}

// ---- start filter ------------------------------------------------------------

__device__ __forceinline__ bool probe(const uint32_t* s_filter, uint32_t slot)
{
    return (s_filter[slot >> 5] >> (slot & 31u)) & 1u;
}

// Bit j set = start j of this thread may report.  First probe on all 16
// starts (branch-free), second probe only on the survivors of the first.
template <int KW>
__device__ __forceinline__ uint32_t filter_mask(const TrieView& t, const uint8_t* s_text, const uint32_t* s_filter,
                                                uint32_t base, uint32_t valid)
{
    if (KW == 0) return valid;
    const uint4 q = *reinterpret_cast<const uint4*>(s_text + base);
    const uint2 r = *reinterpret_cast<const uint2*>(s_text + base + 16);
    const uint32_t w[6] = {q.x, q.y, q.z, q.w, r.x, r.y};
    const uint32_t k = t.filter_k, bits = t.filter_bits;
    const uint32_t m32 = k >= 4 ? 0xFFFFFFFFu : ((1u << (8 * k)) - 1u);
    const uint32_t mhi = k >= 8 ? 0xFFFFFFFFu : (k > 4 ? ((1u << (8 * (k - 4))) - 1u) : 0u);
    auto key32 = [&](int j) { return __funnelshift_r(w[j >> 2], w[(j >> 2) + 1], 8 * (j & 3)) & m32; };
    auto key64 = [&](int j) {
        const uint32_t lo = __funnelshift_r(w[j >> 2], w[(j >> 2) + 1], 8 * (j & 3));
        const uint32_t hi = __funnelshift_r(w[(j >> 2) + 1], w[(j >> 2) + 2], 8 * (j & 3)) & mhi;
        return (uint64_t(hi) << 32) | lo;
    };
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < int(kPerThread); ++j) {
        const uint32_t slot = KW == 1 ? filter_slot32(key32(j), bits) : filter_slot64(key64(j), bits);
        m |= uint32_t(probe(s_filter, slot)) << j;
    }
    m &= valid;
    if (m && t.filter_hashes > 1) {
        uint32_t m2 = 0;
#pragma unroll
        for (int j = 0; j < int(kPerThread); ++j) {
            if ((m >> j) & 1u) {
                const uint32_t slot = KW == 1 ? filter_slot32b(key32(j), bits) : filter_slot64b(key64(j), bits);
                m2 |= uint32_t(probe(s_filter, slot)) << j;
            }
        }
        m = m2;
    }
    return m;
}

// ---- block scan (exclusive) over one 32-bit value per thread ----------------

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t& total)
{
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= uint32_t(d)) incl += u;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t x = lane < kWarps ? s_warp[lane] : 0u;
        uint32_t xi = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, xi, d);
            if (lane >= uint32_t(d)) xi += u;
        }
        if (lane < kWarps) s_warp[lane] = xi - x;
        if (lane == kWarps - 1) s_warp[kWarps] = xi;
    }
    __syncthreads();
    total = s_warp[kWarps];
    return s_warp[warp] + incl - v;
}

// ---- the kernel ----------------------------------------------------------------

struct SmemLayout {
    uint32_t filter_bytes, sym_bytes;
    __host__ __device__ static constexpr uint32_t text_bytes() { return 2 * kSmemText; }
    __host__ __device__ static constexpr uint32_t queue_bytes() { return kTile * 2; }
};

template <bool GROUPED, bool IDENT, int KW>
__global__ void __launch_bounds__(kThreads, 2) pfac_scan_kernel(const __grid_constant__ ScanArgs a)
{
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t fwords = KW ? a.trie.filter_words : 0u;
    uint8_t* s_text0 = smem;                                       // 2 x kSmemText
    uint16_t* s_queue = reinterpret_cast<uint16_t*>(smem + 2 * kSmemText);
    uint32_t* s_filter = reinterpret_cast<uint32_t*>(smem + 2 * kSmemText + 2 * kTile);
    uint16_t* s_sym = reinterpret_cast<uint16_t*>(s_filter + fwords);
    __shared__ uint64_t s_bar[2];
    __shared__ uint32_t s_warp[kWarps + 1];
    __shared__ unsigned long long s_tile[2], s_slot;

    const uint32_t tid = threadIdx.x;
    const TrieView& t = a.trie;
    for (uint32_t i = tid; i < fwords; i += kThreads) s_filter[i] = __ldg(t.filter + i);
    if (!IDENT)
        for (uint32_t i = tid; i < 256; i += kThreads) s_sym[i] = __ldg(t.symtab + i);

    const uint64_t avail16 = (a.n_avail + 15) & ~15ull;
    // Thread 0 keeps one claim in flight beyond the two buffered tiles, so the
    // atomic's latency never sits on the critical path.  Every CTA ends with
    // exactly three failed claims (two buffers + the pending one): the host
    // advances its counter base by n_tiles + 3 * grid per launch.
    unsigned long long pending = 0;
    auto issue = [&](uint32_t buf) {
        const unsigned long long tile = pending - a.tile_base;
        pending = atomicAdd(a.tile_ctr, 1ull);
        s_tile[buf] = tile;
        if (tile < a.n_tiles) {
            const uint64_t lo = tile * kTile;
            const uint32_t n = uint32_t(min(uint64_t(kSmemText), avail16 - lo));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_load(s_text0 + buf * kSmemText, a.text + lo, n, &s_bar[buf]);
        }
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        pending = atomicAdd(a.tile_ctr, 1ull);
        issue(0);
        issue(1);
    }
    __syncthreads();

    const uint64_t me = t.min_emit;
    const uint64_t start_end = a.n_avail >= me ? min(a.n_own, a.n_avail - me + 1) : 0;
    uint32_t parity[2] = {0, 0};

    for (uint32_t buf = 0;; buf ^= 1) {
        const unsigned long long tile = s_tile[buf];
        if (tile >= a.n_tiles) break;
        mbar_wait(&s_bar[buf], parity[buf]);
        parity[buf] ^= 1;
        const uint8_t* s_text = s_text0 + buf * kSmemText;
        const uint64_t lo = tile * kTile;
        const TileCtx c{s_text, s_sym, lo, uint32_t(min(uint64_t(kSmemText), avail16 - lo))};

        // (b) filter this thread's 16 starts
        const uint64_t o0 = lo + uint64_t(tid) * kPerThread;
        uint32_t valid = 0;
        if (o0 < start_end) {
            const uint64_t r = start_end - o0;
            valid = r >= kPerThread ? 0xFFFFu : ((1u << r) - 1u);
        }
        const uint32_t mask = valid ? filter_mask<KW>(t, s_text, s_filter, tid * kPerThread, valid) : 0u;

        // (c) ordered compaction of survivors
        uint32_t q_total;
        uint32_t q_at = block_exclusive_scan(__popc(mask), s_warp, q_total);
        for (uint32_t m = mask; m; m &= m - 1) s_queue[q_at++] = uint16_t(tid * kPerThread + __ffs(m) - 1);
        __syncthreads();

        // (d) walk an even share of the queue
        const uint32_t per = (q_total + kThreads - 1) / kThreads;
        const uint32_t e0 = min(q_total, tid * per), e1 = min(q_total, e0 + per);
        Sink sink;
        for (uint32_t e = e0; e < e1; ++e) walk<GROUPED, IDENT>(a, c, lo + s_queue[e], sink);

        // (e) order the tile's records and reserve its staging slice
        uint32_t tile_total;
        const uint32_t my_at = block_exclusive_scan(sink.n, s_warp, tile_total);
        if (tid == 0) {
            const unsigned long long slot = tile_total ? atomicAdd(a.stage_cursor, (unsigned long long)tile_total) : 0;
            s_slot = slot;
            a.tile_count[tile] = tile_total;
            a.tile_slot[tile] = slot;
        }
        __syncthreads();
        if (sink.n) {
            const uint64_t at = s_slot + my_at;
            uint4* stage = reinterpret_cast<uint4*>(a.stage);
            if (at < a.cap) stage[at] = sink.r0;
            if (sink.n > 1 && at + 1 < a.cap) stage[at + 1] = sink.r1;
            if (sink.n > kRegRecords) { // rare: re-walk and write the rest directly
                Sink w;
                w.dst = a.stage;
                w.at = at + kRegRecords;
                w.cap = a.cap;
                w.skip = kRegRecords;
                for (uint32_t e = e0; e < e1; ++e) walk<GROUPED, IDENT>(a, c, lo + s_queue[e], w);
            }
        }
        __syncthreads(); // buffer, queue and s_slot free again
        if (tid == 0) issue(buf);
    }

    // phase 2: exclusive scan of per-tile counts, chunked by CTA
    cg::grid_group grid = cg::this_grid();
    grid.sync();
    if (blockIdx.x == 0 && tid == 0) *a.stage_cursor = 0; // ready for the next launch
    const uint64_t nt = a.n_tiles, chunk = (nt + gridDim.x - 1) / gridDim.x;
    const uint64_t c0 = min(nt, uint64_t(blockIdx.x) * chunk), c1 = min(nt, c0 + chunk);
    {
        uint32_t s = 0;
        for (uint64_t i = c0 + tid; i < c1; i += kThreads) s += a.tile_count[i];
        uint32_t tot;
        block_exclusive_scan(s, s_warp, tot);
        if (tid == 0) a.chunk_sum[blockIdx.x] = tot;
    }
    grid.sync();
    {
        unsigned long long base = 0;
        for (uint32_t b = 0; b < blockIdx.x; ++b) base += a.chunk_sum[b]; // all threads, L1-cached
        // scan the chunk in rounds of kThreads tiles
        for (uint64_t r0 = c0; r0 < c1; r0 += kThreads) {
            const uint64_t i = r0 + tid;
            const uint32_t v = i < c1 ? a.tile_count[i] : 0u;
            uint32_t tot;
            const uint32_t ex = block_exclusive_scan(v, s_warp, tot);
            if (i < c1) a.tile_first[i] = base + ex;
            base += tot;
            __syncthreads();
        }
        if (c1 == nt && c0 < c1 && tid == 0) *a.total = base;
        if (nt == 0 && blockIdx.x == 0 && tid == 0) *a.total = 0;
    }
    grid.sync();

    // phase 3: staged slices -> final positions (one tile per thread)
    const unsigned long long total = *a.total;
    if (total > a.cap) return; // host re-runs with the exact size
    for (uint64_t i = uint64_t(blockIdx.x) * kThreads + tid; i < nt; i += uint64_t(gridDim.x) * kThreads) {
        const uint32_t n = a.tile_count[i];
        if (!n) continue;
        const uint4* src = reinterpret_cast<const uint4*>(a.stage) + a.tile_slot[i];
        uint4* dst = reinterpret_cast<uint4*>(a.out) + a.tile_first[i];
        for (uint32_t k = 0; k < n; ++k) dst[k] = src[k];
    }
}

// Evicts the text from L2 between timed iterations when it would fit there.
__global__ void l2_flush_kernel(uint4* buf, size_t n16, uint32_t salt)
{
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
        buf[i] = make_uint4(salt, uint32_t(i), 0u, 0u);
}

} // namespace hfb::gpu

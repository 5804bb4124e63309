// filter_kernel.cuh -- the filter passes of the two-pass scan pipeline.
//
// Reference semantics: none of their own -- they only discard start offsets
// that cannot report (a conservative pre-filter of scan.cpp:82-87, where
// every offset starts a walk).  Every start that survives is walked by the
// second pass (pfac_scan_kernel<..., CANDS = true>), which produces the
// records.
//
// Why separate kernels: a filter needs ~60 registers, the walk ~120.  In one
// kernel the walk's register budget caps the SM at 16 warps, and the filter
// (random shared-memory probes, short dependent chains) is latency bound at
// 16 warps.  Alone it runs 32 warps per SM.
//
// Forms: pfac_pair_filter_kernel (pair probes, in-lane
// second level, optional L2 third level), pfac_l2_filter_kernel (single
// probe + L2 bitmap for saturated dictionaries), pfac_pack_symbols_kernel +
// pfac_symbol_filter_kernel (packed symbol keys for sigma <= 4).  All share
// the tiling (8192-start tiles round-robin over warps, 512-start chunks of 16
// consecutive starts per lane) and the output: survivors in start order in
// the warp's region of the candidate buffer (u16 tile offset + first 4 text
// bytes), a count and slot per tile.
#pragma once

#include <cuda_runtime.h>

#include "layout.hpp"

namespace hfb::gpu {

#ifndef HFB_FWARPS
#define HFB_FWARPS 32
#endif
constexpr uint32_t kFWarps = HFB_FWARPS;
constexpr uint32_t kFThreads = kFWarps * 32;
constexpr uint32_t kFChunk = 512;                     // bytes per warp chunk (16 per lane)
constexpr uint32_t kFChunks = 4;                      // chunks per step
constexpr uint32_t kFStep = kFChunk * kFChunks;       // 2 KiB
constexpr uint32_t kFTile = 8192;                     // == kTile of scan_kernel.cuh

struct FilterArgs {
    const uint32_t* table;   // pair table, 2^wb words
    uint32_t table_words;
    uint32_t pair_shift;     // 32 - wb
    const uint8_t* text;     // 16-byte aligned, readable up to round_up(n_avail, 16) + 16
    uint64_t n_avail;        // bytes of text
    uint64_t start_end;      // starts [0, start_end) may report
    uint64_t n_tiles;
    uint16_t* cand;          // gridDim.x * kFWarps regions of cand_cap entries
    uint32_t* cand_key;      // same layout: the survivor's first 4 text bytes
    uint64_t cand_cap;
    uint32_t* tile_ccount;
    uint32_t* tile_cslot;
    unsigned long long* cand_need; // max entries any warp needed (overflow sizing)
    // symbol form: k symbols per key; single + L2 form: k bytes
    uint32_t filter_k;
    const uint32_t* table2;  // single + L2 form: the 2^table2_bits-bit bitmap in global memory
    uint32_t table2_bits;
    const uint32_t* packed;  // symbol form: the text packed by pfac_pack_symbols_kernel
};

__device__ __forceinline__ uint32_t f_lds(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// First level over one 16-start lane slice: w[0..3] its bytes, w[4] the next 4.
// Bit j = start j passed its first role (layout.hpp, pair form).
__device__ __forceinline__ uint32_t f_pair_level1(const uint32_t (&w)[5], uint32_t tbase, uint32_t shift)
{
    uint32_t m0 = 0, m1 = 0; // two independent chains, MSB-first
#pragma unroll
    for (int i = 1; i < 16; i += 2) {
        auto win = [&](int n) -> uint32_t {
            return (n & 3) ? __funnelshift_r(w[n >> 2], w[(n >> 2) + 1], 8 * (n & 3)) : w[n >> 2];
        };
        const uint32_t mid = win(i), a = win(i - 1), b = win(i + 3);
        const uint32_t word = f_lds(tbase + (((mid * kPairMul) >> shift) << 2));
        uint32_t& m = i < 8 ? m0 : m1;
        m = __funnelshift_l(__funnelshift_l(0u, word, a), m, 1); // start i - 1 (role A)
        m = __funnelshift_l(__funnelshift_l(0u, word, b), m, 1); // start i (role B)
    }
    return __brev((m0 << 24) | (m1 << 16)); // start j at bit j
}

// ---- pair form -------------------------------------------------------------------
//
// Per 2 KiB step a lane loads its 4 slices (16 B each, coalesced), the step
// is staged contiguously in shared memory, and the first level (8 pair
// probes per slice) gives 16 bits per slice.  The second level is done by
// each lane on its own first-level survivors, reading their bytes back from
// the staged step: one loop over the lane's 64 starts, so a step costs
// max-over-lanes(survivors) iterations of a ~32-instruction loop.  (A queue form that redistributed survivors to full
// 32-lane rounds spent 36% of the pass building the queue and was measured
// 0.5-8% slower: c3, c4 sigma=256, c5 10k.)  Final survivors (~0.1%) are
// placed in start order by one ballot per chunk.
constexpr uint32_t kPStage = kFStep + 16;             // staged step + the word after it
constexpr uint32_t kPWarpSmem = kPStage;

__device__ __forceinline__ uint32_t f_pair_probe(const uint32_t* __restrict__ tab, uint32_t mid, uint32_t shift)
{
    return tab[(mid * kPairMul) >> shift];
}

// L2: the image has an L2-resident third level (dense pair survivors); a
// separate instantiation keeps the common case's code unchanged.
template <bool L2>
__global__ void __launch_bounds__(kFThreads, 1) pfac_pair_filter_kernel(const __grid_constant__ FilterArgs a)
{
    extern __shared__ __align__(128) uint8_t fsmem[];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint32_t* s_tab = reinterpret_cast<uint32_t*>(fsmem);
    for (uint32_t i = tid; i < a.table_words; i += kFThreads) s_tab[i] = __ldg(a.table + i);
    __syncthreads();
    uint8_t* stage = fsmem + size_t(a.table_words) * 4 + warp * kPWarpSmem;
    const uint32_t stage_s = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    const uint32_t tbase = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));

    const uint32_t gw = blockIdx.x * kFWarps + warp, W = gridDim.x * kFWarps;
    const uint32_t shift = a.pair_shift;
    const uint64_t avail16 = (a.n_avail + 15) & ~15ull;
    uint16_t* region = a.cand + uint64_t(gw) * a.cand_cap;
    uint32_t* keys = a.cand_key + uint64_t(gw) * a.cand_cap;
    const uint32_t cap = uint32_t(min(a.cand_cap, uint64_t(0xFFFFFFFFu)));
    uint32_t cursor = 0;
    const uint32_t below = (1u << lane) - 1u;
    const uint32_t my = stage_s + 16u * lane; // this lane's 16 bytes of chunk 0

    auto load = [&](uint64_t at) -> uint4 {
        const uint64_t p = at + 16u * lane;
        return p < avail16 ? __ldg(reinterpret_cast<const uint4*>(a.text + p)) : make_uint4(0u, 0u, 0u, 0u);
    };
    // bytes [so, so + 4) of the staged step
    auto staged4 = [&](uint32_t so) -> uint32_t {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(stage) + (so >> 2);
        uint32_t t;
        asm("prmt.b32.f4e %0, %1, %2, %3;" : "=r"(t) : "r"(w[0]), "r"(w[1]), "r"(so));
        return t;
    };

    for (uint64_t tile = gw; tile < a.n_tiles; tile += W) {
        const uint64_t lo = tile * kFTile;
        const uint32_t slot = cursor;
        const uint32_t rem = a.start_end > lo ? uint32_t(min(a.start_end - lo, uint64_t(kFTile))) : 0u;
        const uint32_t steps = (rem + kFStep - 1) / kFStep;
        uint4 nxt[kFChunks];
        if (steps) {
#pragma unroll
            for (uint32_t b = 0; b < kFChunks; ++b) nxt[b] = load(lo + b * kFChunk);
        }
        for (uint32_t s = 0; s < steps; ++s) {
            const uint64_t sbase = lo + uint64_t(s) * kFStep;
            uint4 cur[kFChunks];
#pragma unroll
            for (uint32_t b = 0; b < kFChunks; ++b) cur[b] = nxt[b];
            // the next step's loads: issued after this step's second level, so
            // their registers are not live across it (+2% at c3 against issuing
            // them one step ahead at the top of the step)
            auto prefetch = [&]() {
                if (s + 1 < steps) {
                    const uint64_t nb = sbase + kFStep;
                    if (nb + kFStep <= avail16) { // warp-uniform: the whole next step is in the buffer
                        const uint4* src = reinterpret_cast<const uint4*>(a.text + nb) + lane;
#pragma unroll
                        for (uint32_t b = 0; b < kFChunks; ++b) nxt[b] = __ldg(src + b * (kFChunk / 16));
                    } else {
#pragma unroll
                        for (uint32_t b = 0; b < kFChunks; ++b) nxt[b] = load(nb + b * kFChunk);
                    }
                }
            };
            // the 4 bytes after the step (8 with the third level: its keys
            // reach 8 bytes past a start)
            uint2 tail = make_uint2(0u, 0u);
            if (lane == 31 && sbase + kFStep < avail16) {
                if (L2) tail = __ldg(reinterpret_cast<const uint2*>(a.text + sbase + kFStep));
                else tail.x = __ldg(reinterpret_cast<const uint32_t*>(a.text + sbase + kFStep));
            }
            __syncwarp(); // the previous step's staged bytes are no longer read
#pragma unroll
            for (uint32_t b = 0; b < kFChunks; ++b)
                *reinterpret_cast<uint4*>(stage + b * kFChunk + 16u * lane) = cur[b];
            if (lane == 31) {
                if (L2) *reinterpret_cast<uint2*>(stage + kFStep) = tail;
                else *reinterpret_cast<uint32_t*>(stage + kFStep) = tail.x;
            }
            __syncwarp();

            const bool full = (s + 1) * kFStep <= rem; // warp-uniform: every start of the step may report
            uint32_t m01 = 0, m23 = 0; // first-level survivors, 16 bits per chunk
#pragma unroll
            for (uint32_t b = 0; b < kFChunks; ++b) {
                uint32_t ov; // the 4 bytes after this lane's 16
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(ov) : "r"(my + b * kFChunk + 16u));
                const uint32_t w[5] = {cur[b].x, cur[b].y, cur[b].z, cur[b].w, ov};
                uint32_t m = f_pair_level1(w, tbase, shift);
                if (!full) {
                    const int32_t r = int32_t(rem) - int32_t(s * kFStep + b * kFChunk + 16u * lane);
                    m &= r >= 16 ? 0xFFFFu : (r > 0 ? (1u << r) - 1u : 0u);
                }
                if (b == 0) m01 = m;
                else if (b == 1) m01 |= m << 16;
                else if (b == 2) m23 = m;
                else m23 |= m << 16;
            }
            if (!__any_sync(0xFFFFFFFFu, m01 | m23)) {
                prefetch();
                continue;
            }

            // second level, in-lane: the other role of each first-level
            // survivor, highest bit first (bit j of a word = chunk j/16,
            // position j%16 of the lane's slice; m01: chunks 0-1, m23: 2-3).
            // Failing bits are cleared.
            {
                // loop constants kept opaque, so they stay in registers
                uint32_t k_one, k_mul, k_shift;
                asm("mov.u32 %0, 1;" : "=r"(k_one));
                asm("mov.u32 %0, %1;" : "=r"(k_mul) : "n"(kPairMul));
                asm("mov.u32 %0, %1;" : "=r"(k_shift) : "r"(shift));
                // one second-level test of bit j (0..31) of the mask whose
                // chunk pair starts at `base`; returns bit j if it fails
                auto test = [&](uint32_t base, uint32_t j, uint32_t bit, uint32_t& fail) {
                    const uint32_t at = base + j + (j >> 4) * (kFChunk - 16u); // + chunk * 512 + position
                    uint32_t w0, w1, t;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w0) : "r"(at & ~3u));
                    asm volatile("ld.shared.u32 %0, [%1+4];" : "=r"(w1) : "r"(at & ~3u));
                    asm("prmt.b32.f4e %0, %1, %2, %3;" : "=r"(t) : "r"(w0), "r"(w1), "r"(at)); // p0 p1 p2 p3
                    // odd starts passed role B and test A: H(p1 p2 p3), bit p0;
                    // even ones test B: H(p0 p1 p2), bit p3.  sh = 8 for odd j:
                    // mid = t >> sh, and the amount t >> (24 + sh) mod 32.
                    const uint32_t sh = (j << 3) & 8u;
                    const uint32_t mid = t >> sh, amt = __funnelshift_r(t, 0u, sh + 24u);
                    const uint32_t word = f_lds(tbase + (((mid * k_mul) >> k_shift) << 2));
                    // fail |= bit unless the tested bit (now the sign) is set:
                    // one arithmetic shift and one LOP3 instead of a compare,
                    // a select and an OR
                    uint32_t sgn;
                    asm("shr.s32 %0, %1, 31;" : "=r"(sgn) : "r"(__funnelshift_l(0u, word, amt)));
                    asm("lop3.b32 %0, %1, %2, %3, 0xF4;" : "=r"(fail) : "r"(fail), "r"(bit), "r"(sgn)); // fail | (bit & ~sgn)
                };
                const uint32_t base01 = stage_s + 16u * lane;
                uint32_t fail01 = 0, fail23 = 0;
                if constexpr (!L2) {
                    // one loop over both words (m23 first): a step costs the
                    // maximum over lanes of the lane's survivors, not the sum of
                    // the two words' maxima.  When the current word runs out the
                    // other one takes its place (predicated, no branch): 32
                    // instructions per iteration against 24, for ~6.1 iterations
                    // per step against ~7.8 at c3 (+0.7-2.7% on c3, c4 sigma=64/256,
                    // c5 1k/10k).  The third-level instantiation keeps two loops
                    // (c5 100k: +4.5% with two, +0.6% with one).
                    uint32_t x = m23, fail = 0, f23 = 0, base = base01 + 2u * kFChunk;
                    bool second = false;
                    if (!x) x = m01, second = true, base = base01;
                    while (x) {
                        uint32_t j;
                        asm("bfind.u32 %0, %1;" : "=r"(j) : "r"(x)); // highest set bit
                        const uint32_t bit = k_one << j;
                        x ^= bit;
                        test(base, j, bit, fail);
                        if (!x && !second) x = m01, f23 = fail, fail = 0, base = base01, second = true;
                    }
                    fail23 = second ? f23 : fail;
                    fail01 = second ? fail : 0u;
                } else {
#pragma unroll
                    for (uint32_t half = 0; half < 2; ++half) {
                        const uint32_t base = base01 + half * 2u * kFChunk;
                        uint32_t fail = 0;
                        for (uint32_t x = half ? m23 : m01; x;) {
                            uint32_t j;
                            asm("bfind.u32 %0, %1;" : "=r"(j) : "r"(x)); // highest set bit
                            const uint32_t bit = k_one << j;
                            x ^= bit;
                            test(base, j, bit, fail);
                        }
                        if (half) fail23 = fail;
                        else fail01 = fail;
                    }
                }
                m01 &= ~fail01;
                m23 &= ~fail23;
            }
            // third level (dictionaries whose pair survivors are dense, e.g. c5
            // 100k: 3.6% of starts): both bits of the start's k-byte key in the
            // L2-resident bitmap (image.cpp), four survivors' loads in flight
            // per round, before the survivors are written out.  Conservative:
            // it only removes starts no dictionary path begins with.
            if (L2 && __any_sync(0xFFFFFFFFu, m01 | m23)) {
                const uint32_t sh2 = 32u - a.table2_bits, base = 16u * lane;
                const uint32_t k = a.filter_k;
                const uint32_t mhi = k >= 8 ? 0xFFFFFFFFu : (k > 4 ? ((1u << (8 * (k - 4))) - 1u) : 0u);
                uint64_t left = (uint64_t(m23) << 32) | m01, fail = 0;
                while (__any_sync(0xFFFFFFFFu, left != 0)) {
                    uint32_t w2[4], h2[4], jj[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        w2[r] = 0xFFFFFFFFu, h2[r] = 0u, jj[r] = 64u;
                        if (left) {
                            uint32_t j;
                            asm("bfind.u64 %0, %1;" : "=r"(j) : "l"(left));
                            left ^= 1ull << j;
                            const uint32_t so = base + (j & 15u) + (j >> 4) * kFChunk;
                            uint32_t key = staged4(so);
                            if (mhi) key += (staged4(so + 4) & mhi) * 0x85EBCA77u; // filter_fold
                            const uint32_t h = filter2_hash(key);
                            h2[r] = ((h >> sh2) & 31u) | ((h & 31u) << 8);
                            w2[r] = __ldg(a.table2 + ((h >> sh2) >> 5));
                            jj[r] = j;
                        }
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (jj[r] < 64u && !((w2[r] >> (h2[r] & 31u)) & (w2[r] >> (h2[r] >> 8)) & 1u))
                            fail |= 1ull << jj[r];
                }
                m01 &= ~uint32_t(fail);
                m23 &= ~uint32_t(fail >> 32);
            }
            prefetch();
            if (!__any_sync(0xFFFFFFFFu, m01 | m23)) continue;
            const uint32_t n01 = __popc(m01), n23 = __popc(m23);
            // final survivors in start order (chunk, lane, position).  Common
            // case (~90% of steps at c3): at most one per lane, placed by one
            // ballot per chunk.
            if (!__any_sync(0xFFFFFFFFu, n01 + n23 > 1)) {
                const uint32_t c0 = __ballot_sync(0xFFFFFFFFu, m01 & 0xFFFFu), c1 = __ballot_sync(0xFFFFFFFFu, m01 >> 16);
                const uint32_t c2 = __ballot_sync(0xFFFFFFFFu, m23 & 0xFFFFu), c3 = __ballot_sync(0xFFFFFFFFu, m23 >> 16);
                const uint32_t p1 = __popc(c0), p2 = p1 + __popc(c1), p3 = p2 + __popc(c2);
                if (m01 | m23) {
                    const uint32_t j = m01 ? __ffs(m01) - 1 : 32u + __ffs(m23) - 1; // bit in the lane's 64
                    const uint32_t b = j >> 4;
                    const uint32_t bal = b == 0 ? c0 : (b == 1 ? c1 : (b == 2 ? c2 : c3));
                    const uint32_t at = cursor + (b == 0 ? 0u : (b == 1 ? p1 : (b == 2 ? p2 : p3))) + __popc(bal & below);
                    const uint32_t so = b * kFChunk + 16u * lane + (j & 15u);
                    if (at < cap) {
                        region[at] = uint16_t(s * kFStep + so);
                        keys[at] = staged4(so);
                    }
                }
                cursor += p3 + __popc(c3);
                continue;
            }
            // otherwise one warp scan of the lane's four per-chunk counts
            // packed in 8-bit fields (exact while every lane has at most 7
            // survivors in the step)
            const uint32_t cnt = (__popc(m01 & 0xFFFFu)) | ((n01 - __popc(m01 & 0xFFFFu)) << 8) |
                                 (__popc(m23 & 0xFFFFu) << 16) | ((n23 - __popc(m23 & 0xFFFFu)) << 24);
            if (__any_sync(0xFFFFFFFFu, n01 + n23 > 7u)) {
                // dense step: chunk by chunk, one scan each
#pragma unroll
                for (uint32_t b = 0; b < kFChunks; ++b) {
                    const uint32_t f = ((b < 2 ? m01 : m23) >> (16u * (b & 1u))) & 0xFFFFu;
                    const uint32_t n = __popc(f);
                    uint32_t incl = n;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                        if (lane >= uint32_t(d)) incl += u;
                    }
                    uint32_t at = cursor + incl - n;
                    for (uint32_t m = f; m; m &= m - 1, ++at) {
                        const uint32_t so = b * kFChunk + 16u * lane + uint32_t(__ffs(m) - 1);
                        if (at < cap) {
                            region[at] = uint16_t(s * kFStep + so);
                            keys[at] = staged4(so);
                        }
                    }
                    cursor += __shfl_sync(0xFFFFFFFFu, incl, 31);
                }
                continue;
            }
            uint32_t incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= uint32_t(d)) incl += u;
            }
            const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
            // byte b: survivors before this lane's chunk-b ones (earlier chunks + earlier lanes)
            const uint32_t pos = incl - cnt + tot * 0x01010100u;
            if (m01 | m23) {
#pragma unroll
                for (uint32_t b = 0; b < kFChunks; ++b) {
                    uint32_t at = cursor + ((pos >> (8u * b)) & 0xFFu);
                    for (uint32_t m = ((b < 2 ? m01 : m23) >> (16u * (b & 1u))) & 0xFFFFu; m; m &= m - 1, ++at) {
                        const uint32_t so = b * kFChunk + 16u * lane + uint32_t(__ffs(m) - 1);
                        if (at < cap) {
                            region[at] = uint16_t(s * kFStep + so);
                            keys[at] = staged4(so);
                        }
                    }
                }
            }
            cursor += (tot * 0x01010101u) >> 24;
        }
        if (lane == 0) {
            a.tile_ccount[tile] = cursor - slot;
            a.tile_cslot[tile] = uint32_t(slot);
        }
    }
    if (lane == 0 && cursor > cap) atomicMax(a.cand_need, (unsigned long long)cursor);
}

// ---- single probe + L2 bitmap (large dictionaries) --------------------------------
//
// For dictionaries whose k-gram set saturates any shared-memory bitmap (c5 at
// 1M patterns: 2^20 bits for ~1M keys pass 61% of random starts), the filter
// pass tests every start against both levels of the single-probe filter
// (layout.hpp): the shared-memory bitmap and the 2^filter2_bits-bit bitmap in
// global memory (16 MiB, L2-resident).  All 16 L2 probes of a lane slice are
// issued before the first is tested (predicated on the first level), so a
// warp has up to 512 L2 loads in flight instead of one dependent chain per
// start; survivors (~1% at 1M patterns) go to the walking pass.
// Key of start j (KW 3: k == 4, KW 2: k in 5..8): the same fold as the host's
// filter_fold.  w[0..5] = the slice's 16 bytes and the next 8.
template <int KW>
__device__ __forceinline__ uint32_t f_key(const uint32_t (&w)[6], int j, uint32_t mhi)
{
    const uint32_t lo = (j & 3) ? __funnelshift_r(w[j >> 2], w[(j >> 2) + 1], 8 * (j & 3)) : w[j >> 2];
    if (KW != 2) return lo;
    const uint32_t hi = ((j & 3) ? __funnelshift_r(w[(j >> 2) + 1], w[(j >> 2) + 2], 8 * (j & 3)) : w[(j >> 2) + 1]) & mhi;
    return lo + hi * 0x85EBCA77u; // filter_fold
}

// L2 bitmap word: random 4-byte reads with no reuse in L1 (HFB_PROBE_NA=1:
// not allocated in L1).
__device__ __forceinline__ uint32_t probe_l2(const uint32_t* p)
{
#if defined(HFB_PROBE_NA) && HFB_PROBE_NA
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

template <int KW>
__global__ void __launch_bounds__(kFThreads, 1) pfac_l2_filter_kernel(const __grid_constant__ FilterArgs a)
{
    extern __shared__ __align__(128) uint8_t fsmem[];
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    uint32_t* s_tab = reinterpret_cast<uint32_t*>(fsmem);
    for (uint32_t i = tid; i < a.table_words; i += kFThreads) s_tab[i] = __ldg(a.table + i);
    __syncthreads();
    const uint32_t words = a.table_words; // filter_l1_word range (any count)
    const uint32_t k = a.filter_k;
    const uint32_t mhi = k >= 8 ? 0xFFFFFFFFu : (k > 4 ? ((1u << (8 * (k - 4))) - 1u) : 0u);
    const uint32_t* l2 = a.table2;
    const uint32_t sh2 = 32u - a.table2_bits;

    const uint32_t gw = blockIdx.x * kFWarps + (tid >> 5), W = gridDim.x * kFWarps;
    const uint64_t avail16 = (a.n_avail + 15) & ~15ull;
    uint16_t* region = a.cand + uint64_t(gw) * a.cand_cap;
    uint32_t* keys = a.cand_key + uint64_t(gw) * a.cand_cap;
    const uint32_t cap = uint32_t(min(a.cand_cap, uint64_t(0xFFFFFFFFu)));
    uint32_t cursor = 0;
    const uint32_t below = (1u << lane) - 1u;
    auto load = [&](uint64_t at) -> uint4 {
        const uint64_t p = at + 16u * lane;
        return p < avail16 ? __ldg(reinterpret_cast<const uint4*>(a.text + p)) : make_uint4(0u, 0u, 0u, 0u);
    };

    for (uint64_t tile = gw; tile < a.n_tiles; tile += W) {
        const uint64_t lo = tile * kFTile;
        const uint32_t slot = cursor;
        const uint32_t rem = a.start_end > lo ? uint32_t(min(a.start_end - lo, uint64_t(kFTile))) : 0u;
        const uint32_t chunks = (rem + kFChunk - 1) / kFChunk;
        uint4 nxt = chunks ? load(lo) : make_uint4(0u, 0u, 0u, 0u);
        for (uint32_t c = 0; c < chunks; ++c) {
            const uint64_t cbase = lo + uint64_t(c) * kFChunk;
            const uint4 cur = nxt;
            if (c + 1 < chunks) nxt = load(cbase + kFChunk);
            // the 8 bytes after the slice: the next lane's first 8, lane 31's
            // from the next chunk (its first lane's load, or memory)
            uint32_t ox = __shfl_sync(0xFFFFFFFFu, cur.x, (lane + 1) & 31u);
            uint32_t oy = __shfl_sync(0xFFFFFFFFu, cur.y, (lane + 1) & 31u);
            const uint32_t nx = __shfl_sync(0xFFFFFFFFu, nxt.x, 0), ny = __shfl_sync(0xFFFFFFFFu, nxt.y, 0);
            if (lane == 31) {
                if (c + 1 < chunks) {
                    ox = nx, oy = ny;
                } else {
                    const uint64_t p = cbase + kFChunk;
                    const uint2 t = p < avail16 ? __ldg(reinterpret_cast<const uint2*>(a.text + p)) : make_uint2(0u, 0u);
                    ox = t.x, oy = t.y;
                }
            }
            const uint32_t w[6] = {cur.x, cur.y, cur.z, cur.w, ox, oy};
            const int32_t r = int32_t(rem) - int32_t(c * kFChunk + 16u * lane);
            const uint32_t valid = r >= 16 ? 0xFFFFu : (r > 0 ? (1u << r) - 1u : 0u);
            // level 1 (shared memory) for the 16 starts, then every level-2
            // probe in flight before the first test
            uint32_t m = 0, w2[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t key = f_key<KW>(w, j, mhi);
                const uint32_t word = s_tab[__umulhi(key * kFilterMul, words)]; // filter_l1_word
                const bool hit = ((valid >> j) & 1u) && int32_t(word << (key & 31u)) < 0;
                const uint32_t h2 = filter2_hash(key), s2 = h2 >> sh2;
                // both of the key's bits in its L2 word (image.cpp, mode 4)
                w2[j] = hit ? probe_l2(l2 + (s2 >> 5)) : 0u;
                w2[j] = (w2[j] >> (s2 & 31u)) & (w2[j] >> (h2 & 31u));
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) m |= (w2[j] & 1u) << j;
            if (!__any_sync(0xFFFFFFFFu, m)) continue;
            // survivors in start order (chunk, lane, j)
            const uint32_t n = __popc(m);
            uint32_t at;
            if (!__any_sync(0xFFFFFFFFu, n > 1)) {
                at = cursor + __popc(__ballot_sync(0xFFFFFFFFu, n != 0) & below);
            } else {
                uint32_t incl = n;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                    if (lane >= uint32_t(d)) incl += u;
                }
                at = cursor + incl - n;
            }
            const uint32_t first = c * kFChunk + 16u * lane; // tile offset of the slice
            for (uint32_t x = m; x; x &= x - 1, ++at) {
                const int j = __ffs(x) - 1;
                if (at < cap) { // (rare: re-read the first 4 bytes rather than index w[] dynamically)
                    const uint64_t pos = lo + first + uint32_t(j);
                    const uint32_t* tp = reinterpret_cast<const uint32_t*>(a.text + (pos & ~3ull));
                    region[at] = uint16_t(first + j);
                    keys[at] = __funnelshift_r(__ldg(tp), __ldg(tp + 1), 8u * uint32_t(pos & 3u));
                }
            }
            cursor += __reduce_add_sync(0xFFFFFFFFu, n);
        }
        if (lane == 0) {
            a.tile_ccount[tile] = cursor - slot;
            a.tile_cslot[tile] = slot;
        }
    }
    if (lane == 0 && cursor > cap) atomicMax(a.cand_need, (unsigned long long)cursor);
}

constexpr uint32_t pair_smem_fixed_bytes() { return kFWarps * kPWarpSmem; }

// ---- symbol-key form (small alphabets) ------------------------------------------

// Packs the text to SB bits per symbol (byte -> alphabet symbol, bytes
// outside the alphabet as symbol 0: only a filter input, the walks re-read
// the bytes), one u32 per 32/SB bytes, LSB-first.
template <int SB>
__global__ void __launch_bounds__(256) pfac_pack_symbols_kernel(const uint8_t* __restrict__ text, uint64_t n_words,
                                                               const uint16_t* __restrict__ symtab,
                                                               uint32_t* __restrict__ packed)
{
    __shared__ uint32_t tab[256];
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
        const uint16_t v = symtab[i];
        tab[i] = v == kNoSym ? 0u : v;
    }
    __syncthreads();
    constexpr uint32_t per = 32 / SB; // bytes per packed word
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < n_words; w += uint64_t(gridDim.x) * blockDim.x) {
        const uint8_t* src = text + w * per;
        uint32_t bytes[per / 4];
        if (per == 8) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(src));
            bytes[0] = v.x, bytes[per / 4 - 1] = v.y;
        } else {
#pragma unroll
            for (uint32_t q = 0; q < per / 16; ++q) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + q);
                bytes[4 * q] = v.x, bytes[4 * q + 1] = v.y, bytes[4 * q + 2] = v.z, bytes[4 * q + 3] = v.w;
            }
        }
        uint32_t key = 0;
#pragma unroll
        for (uint32_t i = 0; i < per; ++i) key |= tab[(bytes[i / 4] >> (8 * (i % 4))) & 0xFFu] << (SB * i);
        packed[w] = key;
    }
}

// Filter pass over packed symbols: lane L of a chunk owns packed word L (32/SB
// starts); the key of start j is the SB*k bits from bit SB*j.  Survivors go to
// the candidate regions with their packed key.
template <int SB>
__global__ void __launch_bounds__(kFThreads, 1) pfac_symbol_filter_kernel(const __grid_constant__ FilterArgs a)
{
    extern __shared__ __align__(128) uint8_t fsmem[];
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    uint32_t* s_tab = reinterpret_cast<uint32_t*>(fsmem);
    for (uint32_t i = tid; i < a.table_words; i += kFThreads) s_tab[i] = __ldg(a.table + i);
    __syncthreads();
    const uint32_t tbase = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
    const uint32_t mask4 = (a.table_words - 1u) << 2;
    const uint32_t kbits = SB * a.filter_k;
    const uint32_t kmask = kbits >= 32 ? 0xFFFFFFFFu : ((1u << kbits) - 1u);
    constexpr uint32_t kPer = 32 / SB;           // starts per packed word (lane)
    constexpr uint32_t kChunk = 32 * kPer;       // starts per warp chunk
    constexpr uint32_t kChunks = kFTile / kChunk;
    const uint32_t* packed = a.packed;

    const uint32_t gw = blockIdx.x * kFWarps + (tid >> 5), W = gridDim.x * kFWarps;
    uint16_t* region = a.cand + uint64_t(gw) * a.cand_cap;
    uint32_t* keys = a.cand_key + uint64_t(gw) * a.cand_cap;
    const uint32_t cap = uint32_t(min(a.cand_cap, uint64_t(0xFFFFFFFFu)));
    uint32_t cursor = 0;
    const uint32_t below = (1u << lane) - 1u;

    for (uint64_t tile = gw; tile < a.n_tiles; tile += W) {
        const uint64_t lo = tile * kFTile;
        const uint32_t slot = cursor;
        const uint32_t rem = a.start_end > lo ? uint32_t(min(a.start_end - lo, uint64_t(kFTile))) : 0u;
        const uint32_t chunks = (rem + kChunk - 1) / kChunk;
        const uint64_t w0 = lo / kPer; // first packed word of the tile
        // each chunk's two words load one chunk ahead (padded array)
        uint32_t n0 = 0, n1 = 0;
        if (chunks) n0 = __ldg(packed + w0 + lane), n1 = __ldg(packed + w0 + lane + 1);
        for (uint32_t c = 0; c < chunks; ++c) {
            const uint32_t a0 = n0, a1 = n1;
            if (c + 1 < chunks) {
                const uint64_t wn = w0 + uint64_t(c + 1) * 32 + lane;
                n0 = __ldg(packed + wn);
                n1 = __ldg(packed + wn + 1);
            }
            uint32_t m0 = 0, m1 = 0;
#pragma unroll
            for (uint32_t j = 0; j < kPer; ++j) {
                const uint32_t key = (j ? __funnelshift_r(a0, a1, SB * j) : a0) & kmask;
                const uint32_t word = f_lds(tbase + (__umulhi(key, kFilterMul) & mask4)); // filter_word(key) * 4
                uint32_t& m = j < kPer / 2 ? m0 : m1;
                m = __funnelshift_l(__funnelshift_l(0u, word, key), m, 1);
            }
            // start j at bit j
            uint32_t keep = __brev((m0 << (32 - kPer / 2)) | (kPer / 2 < 32 ? (m1 << (32 - kPer)) : 0u));
            if (kPer < 32) keep &= (1u << kPer) - 1u;
            const int32_t r = int32_t(rem) - int32_t(c * kChunk + kPer * lane);
            keep &= r >= int32_t(kPer) ? 0xFFFFFFFFu : (r > 0 ? (1u << r) - 1u : 0u);
            if (!__any_sync(0xFFFFFFFFu, keep)) continue;
            // survivors in start order (lane, j): a warp scan of the per-lane counts
            const uint32_t n = __popc(keep);
            uint32_t incl = n;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= uint32_t(d)) incl += u;
            }
            uint32_t at = cursor + incl - n;
            const uint32_t first = c * kChunk + kPer * lane; // tile offset
            for (uint32_t m = keep; m; m &= m - 1, ++at) {
                const uint32_t j = __ffs(m) - 1;
                if (at < cap) {
                    region[at] = uint16_t(first + j);
                    keys[at] = (j ? __funnelshift_r(a0, a1, SB * j) : a0) & kmask;
                }
            }
            cursor += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
        if (lane == 0) {
            a.tile_ccount[tile] = cursor - slot;
            a.tile_cslot[tile] = slot;
        }
    }
    if (lane == 0 && cursor > cap) atomicMax(a.cand_need, (unsigned long long)cursor);
    (void)kChunks;
}

} // namespace hfb::gpu

// dna_kernel.cuh -- the direct-index scan for alphabets of at most 4 symbols
// (filter mode 5; tables in layout.hpp "Direct-index form").
//
// Reference semantics: scan.cpp:20-51 / :69-119 for a trie that accepts
// exactly its dictionary: the records of a start are the dictionary patterns
// that occur there, in (length, id) order (scan.hpp:12-24), for every trie
// state (SURVEY 8(a') 1).  Walks stop at the text end (scan.cpp:26) and bytes
// outside the alphabet kill them (trie.hpp:70-71): a pattern matches only if
// every byte it covers is inside the text and the alphabet.
//
// Two launches per scan:
//   pfac_pack_dna_kernel: text -> 2-bit symbols (16 per u32, LSB first) and
//     one validity bit per byte (32 per u32); memory bound, 0.375 B written
//     per text byte.
//   pfac_dna_kernel (cooperative, one CTA per SM): the table blob goes to
//     shared memory; warps take 8 KiB tiles round-robin.  Per 512-start
//     chunk each lane reads two packed words (its 16 starts + 16 symbols of
//     context) and one validity word, forms the 16 keys of 8 symbols by
//     funnel shifts and tests them in the exact membership bitmap; survivors
//     (real 8-symbol prefixes only: no false positives) queue in start order.
//     A flush gives each lane one queued start: its 32 symbols and 32
//     validity bits come from two L1/L2-hot loads, the key's rank indexes the
//     start's patterns in shared memory, and each is compared 2 bits per
//     symbol at once.  Records are staged per warp and placed in order by
//     place_records (scan_kernel.cuh), as in the other kernels.
#pragma once

#include "scan_kernel.cuh"

namespace hfb::gpu {

constexpr uint32_t kDnaQueue = 1024;      // per-warp queue of tile offsets (>= 2 chunks)
constexpr uint32_t kDnaChunk = 512;       // starts per warp chunk (16 per lane)

// One 32-byte block through the symbol table: 32 codes (two words) and 32
// validity bits; bytes at or past `n` are invalid.
__device__ __forceinline__ void pack_block_table(const uint32_t (&bytes)[8], uint64_t b0, uint64_t n,
                                                 const uint32_t* tab, uint32_t& lo, uint32_t& hi, uint32_t& ok)
{
    lo = hi = ok = 0;
#pragma unroll
    for (uint32_t i = 0; i < 32; ++i) {
        const uint32_t c = b0 + i < n ? tab[(bytes[i / 4] >> (8 * (i % 4))) & 0xFFu] : 0u;
        ok |= (c >> 2) << i;
        if (i < 16) lo |= (c & 3u) << (2 * i);
        else hi |= (c & 3u) << (2 * (i - 16));
    }
}

// Packs text[0, n) into 2-bit symbols and validity bits; words past the text
// (the kernel reads up to 3 packed / 2 validity words ahead) are zero.
// FORMULA: the alphabet's symbol of byte b is ((b >> 1) ^ (b >> 2)) & 3
// (true of "ACGT" and "acgt"; the host checks): four codes per word come from
// three instructions, and a word is valid when every byte equals the
// alphabet byte of its code (one PRMT against the packed alphabet `symw`).
// Words with a byte outside the alphabet (rare) and the last, partial block
// take the table path.
template <bool FORMULA>
__global__ void __launch_bounds__(256) pfac_pack_dna_kernel(const uint8_t* __restrict__ text, uint64_t n,
                                                           const uint16_t* __restrict__ symtab, uint32_t symw,
                                                           uint32_t* __restrict__ packed,
                                                           uint32_t* __restrict__ valid, uint64_t vwords)
{
    __shared__ uint32_t tab[256]; // symbol + 4 (valid), or 0 (outside the alphabet)
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
        const uint16_t v = symtab[i];
        tab[i] = v == kNoSym ? 0u : 4u + (v & 3u);
    }
    __syncthreads();
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < vwords; w += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t b0 = w * 32;
        uint32_t bytes[8] = {};
        if (b0 < n) { // the text buffer is readable up to round_up(n, 16) + 16 >= b0 + 32
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(text + b0));
            const uint4 y = __ldg(reinterpret_cast<const uint4*>(text + b0) + 1);
            bytes[0] = x.x, bytes[1] = x.y, bytes[2] = x.z, bytes[3] = x.w;
            bytes[4] = y.x, bytes[5] = y.y, bytes[6] = y.z, bytes[7] = y.w;
        }
        uint32_t lo = 0, hi = 0, ok = 0;
        bool table = !FORMULA || b0 + 32 > n;
        if (!table) {
            bool clean = true;
#pragma unroll
            for (uint32_t q = 0; q < 8; ++q) {
                const uint32_t c = ((bytes[q] >> 1) ^ (bytes[q] >> 2)) & 0x03030303u;
                const uint32_t t = c | (c >> 4);                        // codes of bytes 0,1 / 2,3 in nibbles
                const uint32_t canon = __byte_perm(symw, 0u, __byte_perm(t, 0u, 0x0020u));
                clean = clean && canon == bytes[q];
                const uint32_t u = c | (c >> 6);                        // 4 codes -> bits 0-3, 16-19
                const uint32_t p8 = (u & 0xFu) | ((u >> 12) & 0xF0u);
                if (q < 4) lo |= p8 << (8 * q);
                else hi |= p8 << (8 * (q - 4));
            }
            ok = 0xFFFFFFFFu;
            table = !clean;
        }
        if (table) pack_block_table(bytes, b0, n, tab, lo, hi, ok);
        packed[2 * w] = lo;
        packed[2 * w + 1] = hi;
        valid[w] = ok;
    }
}

constexpr uint32_t dna_smem_bytes(uint32_t keys, uint32_t pats, uint32_t warps)
{
    return ((dna_blob_bytes(keys, pats) + 15) & ~15u) + warps * kDnaQueue * 2;
}

template <uint32_t NW>
__global__ void __launch_bounds__(NW * 32, 1) pfac_dna_kernel(const __grid_constant__ ScanArgs a)
{
    constexpr uint32_t NT = NW * 32;
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ uint32_t s_scr[NW + 1];
    const TrieView& t = a.trie;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t nk = t.dna_keys, np = t.dna_pats;
    for (uint32_t i = tid; i < t.dna_words; i += NT) reinterpret_cast<uint32_t*>(dsm)[i] = __ldg(t.dna + i);
    const uint32_t* s_bits = reinterpret_cast<const uint32_t*>(dsm);
    const uint16_t* s_wrank = reinterpret_cast<const uint16_t*>(dsm + kDnaWrankOff);
    const uint16_t* s_first = reinterpret_cast<const uint16_t*>(dsm + kDnaFirstOff);
    const uint64_t* s_sym = reinterpret_cast<const uint64_t*>(dsm + dna_sym_off(nk));
    const uint32_t* s_meta = reinterpret_cast<const uint32_t*>(dsm + dna_meta_off(nk, np));
    uint16_t* q = reinterpret_cast<uint16_t*>(dsm + ((dna_blob_bytes(nk, np) + 15) & ~15u)) + warp * kDnaQueue;
    __syncthreads();

    const uint32_t* P = a.packed; // 16 symbols per word
    const uint32_t* V = a.valid;  // 32 validity bits per word
    const uint64_t start_end = a.n_avail >= kDnaK ? min(a.n_own, a.n_avail - kDnaK + 1) : 0;
    const uint32_t gw = blockIdx.x * NW + warp, W = gridDim.x * NW;
    hepfac_match_t* region = a.stage + uint64_t(gw) * a.warp_cap;
    uint64_t cursor = 0;

    // One queued start per lane: compare its patterns, stage its records.
    auto flush = [&](uint64_t lo, uint32_t n) {
        for (uint32_t r0 = 0; r0 < n; r0 += 32) {
            const uint32_t e = r0 + lane;
            uint64_t s = 0;
            uint32_t f0 = 0, mask = 0;
            if (e < n) {
                s = lo + q[e];
                const uint64_t wi = s >> 4;
                const uint32_t sh = 2u * uint32_t(s & 15u);
                const uint32_t x0 = __ldg(P + wi), x1 = __ldg(P + wi + 1), x2 = __ldg(P + wi + 2);
                const uint64_t vi = s >> 5;
                // ~validity of bytes [s, s + 32): 0 bits = inside the alphabet
                // and the text (the pack pass leaves bytes past the end invalid)
                const uint32_t nv = ~__funnelshift_r(__ldg(V + vi), __ldg(V + vi + 1), uint32_t(s & 31u));
                const uint32_t tlo = __funnelshift_r(x0, x1, sh), thi = __funnelshift_r(x1, x2, sh);
                const uint32_t key = tlo & 0xFFFFu;
                const uint32_t word = s_bits[key >> 5];
                const uint32_t r = s_wrank[key >> 5] + __popc(word & __funnelshift_lc(~0u, 0u, key & 31u));
                f0 = s_first[r];
                const uint32_t cnt = s_first[r + 1] - f0;
                // pattern k matches: its 2-bit symbols equal the text's and
                // its len bytes are valid (len in [8, 32])
                auto test = [&](uint32_t k) -> uint32_t {
                    const uint2 sym = *reinterpret_cast<const uint2*>(s_sym + f0 + k);
                    const uint32_t len = s_meta[f0 + k] >> 16;
                    const uint32_t mlo = __funnelshift_lc(~0u, 0u, 2 * len);
                    const uint32_t mhi = __funnelshift_lc(~0u, 0u, max(2 * len, 32u) - 32u);
                    const uint32_t diff = ((tlo ^ sym.x) & mlo) | ((thi ^ sym.y) & mhi) | (nv << (32u - len));
                    return diff == 0 ? 1u : 0u;
                };
                mask = test(0); // every candidate has at least one pattern
                for (uint32_t k = 1; k < cnt; ++k) mask |= test(k) << k;
            }
            uint64_t at = cursor;
            uint32_t tot;
            const uint32_t nm = __popc(mask);
            if (!__any_sync(0xFFFFFFFFu, nm > 1)) { // common: at most one record per start
                const uint32_t b = __ballot_sync(0xFFFFFFFFu, nm != 0);
                at += __popc(b & ((1u << lane) - 1u));
                tot = __popc(b);
            } else {
                at += warp_exclusive(nm, lane, tot);
            }
            for (uint32_t m = mask; m; m &= m - 1, ++at) {
                const uint32_t meta = s_meta[f0 + __ffs(m) - 1];
                const uint64_t g = a.g0 + s;
                if (at < a.warp_cap)
                    reinterpret_cast<uint4*>(region)[at] = make_uint4(uint32_t(g), uint32_t(g >> 32), meta >> 16, meta & 0xFFFFu);
            }
            cursor += tot;
        }
        __syncwarp(); // queue reads done before the next writes
    };

    for (uint64_t tile = gw; tile < a.n_tiles; tile += W) {
        const uint64_t lo = tile * kTile;
        const uint64_t slot = cursor;
        const uint32_t rem = start_end > lo ? uint32_t(min(start_end - lo, uint64_t(kTile))) : 0u;
        const uint32_t chunks = (rem + kDnaChunk - 1) / kDnaChunk;
        uint32_t qn = 0;
        for (uint32_t c = 0; c < chunks; ++c) {
            const uint64_t wi = (lo + c * kDnaChunk) / 16 + lane; // this lane's starts: symbols of word wi
            const uint32_t p0 = __ldg(P + wi), p1 = __ldg(P + wi + 1);
            const uint64_t vi = wi >> 1;
            uint32_t v = __funnelshift_r(__ldg(V + vi), __ldg(V + vi + 1), 16u * uint32_t(wi & 1u));
            v &= v >> 1, v &= v >> 2, v &= v >> 4; // bit j: bytes j..j+7 are in the alphabet
            const int32_t r = int32_t(rem) - int32_t(c * kDnaChunk + 16u * lane);
            uint32_t m = 0; // start j's bit enters at 31 and ends at 16 + j
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j) {
                const uint32_t win = j ? __funnelshift_r(p0, p1, 2 * j) : p0; // key = low 16 bits
                const uint32_t word = s_bits[(win >> 5) & 0x7FFu];
                m = __funnelshift_r(m, __funnelshift_r(word, 0u, win), 1); // bit (key & 31) of word
            }
            m = (m >> 16) & v & (r >= 16 ? 0xFFFFu : (r > 0 ? (1u << r) - 1u : 0u));
            if (!__any_sync(0xFFFFFFFFu, m)) continue;
            uint32_t tot;
            const uint32_t ex = warp_exclusive(__popc(m), lane, tot);
            if (qn + tot > kDnaQueue) { // warp-uniform
                flush(lo, qn);
                qn = 0;
            }
            uint32_t at = qn + ex;
            const uint32_t first = c * kDnaChunk + 16u * lane;
            for (uint32_t x = m; x; x &= x - 1) q[at++] = uint16_t(first + __ffs(x) - 1);
            qn += tot;
            __syncwarp();
        }
        if (qn) flush(lo, qn);
        if (lane == 0) {
            a.tile_count[tile] = uint32_t(cursor - slot);
            a.tile_slot[tile] = uint32_t(slot);
        }
    }
    if (lane == 0 && cursor > a.warp_cap) atomicMax(a.warp_need, (unsigned long long)cursor);
    place_records<NW, false>(a, s_scr);
}

} // namespace hfb::gpu

// layout.hpp -- the GPU image of a trie, shared by the host builder (g++)
// and the sm_100a kernels (nvcc).
//
// Node records (node indices are the canonical ones, so a GPU node id is the
// same number hepfac_trie_transition returns):
//   narrow  (sigma <= 32) : uint2 {bitmap, base|flags}                 8 B/node
//   grouped (sigma >  32) : per 64-symbol group g a uint4
//                           {bitmap[2g], bitmap[2g+1], base_g|flags, term_id}
//                           16 B per group: 16/32/64 B for sigma 64/128/256
// base_g = first-child index + popcount of all bitmap words before group g,
// so ONE 16-byte load per text byte resolves a transition (reference Eq. 1,
// trie.hpp:68-79, needs up to 8 dependent word reads at sigma = 256).
// flags: bit 31 terminal, bit 30 carries a verification bucket.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define HFB_HD __host__ __device__ __forceinline__
#else
#define HFB_HD inline
#endif

namespace hfb {

constexpr uint32_t kFlagTerminal = 0x80000000u;
constexpr uint32_t kFlagBucket = 0x40000000u;
constexpr uint32_t kBaseMask = 0x3FFFFFFFu;
constexpr uint32_t kMaxGpuNodes = 0x40000000u;
constexpr uint32_t kNoId = 0xFFFFFFFFu;
constexpr uint32_t kKeep = 0xFFFFFFFEu; // path_id of a node that does not change the walk's path id
constexpr uint16_t kNoSym = 0xFFFFu;
constexpr uint32_t kMaxFilterKey = 8; // bytes hashed by the start filter

// Dictionary key of a matched slice: the slice read as little-endian 32-bit
// words (the last one zero-padded), folded with an odd multiplier, mixed with
// the length.  Word-wise so the GPU hashes 4 bytes per step.
HFB_HD uint64_t slice_step(uint64_t h, uint64_t mul, uint32_t word) { return (h + word + 1) * mul; }
HFB_HD uint64_t slice_key(uint64_t h, uint32_t len) { return h ^ (uint64_t(len) * 0x9E3779B97F4A7C15ull); }
HFB_HD uint64_t mix64(uint64_t k)
{
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

// Start filter, single-probe form: the first k text bytes (little-endian
// packed into a 64-bit key) are folded to 32 bits; the bitmap word comes from
// the high half of a 32x32-bit product (IMAD.HI, then one AND with the word
// mask scaled to bytes), the bit inside the word from the key's low 5 bits
// (the first byte).  Bits are stored MSB-first, so the kernel brings a bit to
// the top with one wrapping funnel shift by the key itself.
constexpr uint32_t kFilterMul = 0x9E3779B1u;
HFB_HD uint32_t filter_fold(uint64_t key)
{
    return uint32_t(key) + uint32_t(key >> 32) * 0x85EBCA77u; // one IMAD in the filter loops
}
HFB_HD uint32_t filter_word(uint32_t key32, uint32_t word_bits)
{
    return uint32_t((uint64_t(key32) * kFilterMul) >> 34) & ((1u << word_bits) - 1u);
}
HFB_HD uint32_t filter_mask_bit(uint32_t key32) { return 0x80000000u >> (key32 & 31u); }
// Filter mode 4's shared-memory level is as large as the L1 data cache
// allows, so its word count is not a power of two: multiply-high range
// reduction.  192 KiB (1.57 M bits) measured best at c5 1M patterns (463
// GB/s, against 384 at 128 KiB): 200 KiB or more moves the shared-memory
// carveout to 228 KiB, and the 28 KiB left to L1 starves the filter pass's
// 16-byte text loads and L2 probes (273-292 GB/s).
#ifndef HFB_L1_KIB
#define HFB_L1_KIB 192
#endif
constexpr uint32_t kL1Words = HFB_L1_KIB * 1024 / 4;
HFB_HD uint32_t filter_l1_word(uint32_t key32, uint32_t words)
{
    return uint32_t((uint64_t(key32 * kFilterMul) * words) >> 32);
}

// Start filter, pair form (k >= 4).  One 32-bit word per 3-byte "middle"
// M = (b1, b2, b3) serves two starts: the start at M's first byte (its 4th
// byte selects the bit: role B) and the start one byte earlier (its 1st byte
// selects the bit: role A), superimposed in the same word.  Text position i
// (odd, inside a 32-start lane slice) probes the middle at i and tests start
// i-1 as role A and start i as role B, so 32 starts cost 16 probes; the other
// role of each survivor is tested afterwards (second level, same table).
// A depth-k path p0 p1 p2 p3 ... sets bit p0 of word H(p1 p2 p3) and bit p3 of
// word H(p0 p1 p2).  H is multiply-shift over the low 24 bits of the packed
// middle (the multiplier's low byte is zero, so the 4th byte drops out).
constexpr uint32_t kPairMul = 0x2545F491u << 8;
HFB_HD uint32_t pair_word(uint32_t middle, uint32_t word_bits) { return (middle * kPairMul) >> (32 - word_bits); }

// Second-level filter (global memory, L2-resident): an independent mixing hash
// of the same folded key into a larger bitmap.  Only first-level survivors
// (about 2%) probe it.  The top bits of the same mix index the jump table.
HFB_HD uint32_t filter2_hash(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}
HFB_HD uint32_t filter2_slot(uint32_t x, uint32_t bits) { return filter2_hash(x) >> (32 - bits); }

// Jump table: every depth-k path string (k = filter_k bytes, little-endian in
// {lo, hi}) -> the node it reaches.  No node above depth k can report
// (k <= min_emit), so a walk may start there instead of at the root.  Cuckoo
// hashing: a key lives in slot jump_slot or jump_slot2, so a lookup is two
// independent loads and no probe loop (a linear-probing loop ran up to the
// slowest lane's chain length per warp).  32-byte slots
//   {lo, hi, node, term, bk_first, bk_count, flags, pend}
// node == kNoId marks an empty slot.  The rest describes the node itself, so a
// walk that starts at the depth limit (truncated tries with k == limit) emits
// without reading the node record or the bucket index: term = its private
// pattern id (kNoId = resolve by key), flags bit 0 terminal, bit 1 bucket,
// pend = the path id a walk carries at the node (image.cpp "path ids").
constexpr uint32_t kJumpWords = 8;
// Inline pattern lists: when at most kJumpExtEntries patterns start with a
// slot's key (flags bit 2 = kJumpInline, the count in bits 3-4), the parallel
// extension table (tables up to 2^kMaxJumpExtBits slots: 256 MiB) holds each as {id,
// len, 24 pattern bytes [inline_skip, +24), zero padded}, in (length, id) order.
// They are every record a start with that key can emit (the trie accepts
// exactly its dictionary), so instead of walking the subtree (or reading the
// terminal and bucket at the depth limit) the start verifies them against the
// text with one extension load.  The cap was 2^19 slots (L2-sized) until c5 at
// 1M patterns (2^21 slots) was measured: its stage-2 DAG walks are HBM round
// trips per byte, and the two dependent loads of slot + list are cheaper
// (469 -> 518 GB/s of text).
constexpr uint32_t kJumpInline = 4u;
constexpr uint32_t kJumpInlineShift = 3u;
constexpr uint32_t kJumpExtEntries = 2;
constexpr uint32_t kJumpExtEntryWords = 8;
constexpr uint32_t kJumpExtBytes = 4 * (kJumpExtEntryWords - 2);
constexpr uint32_t kJumpExtWords = kJumpExtEntries * kJumpExtEntryWords;
#ifndef HFB_MAX_JUMP_EXT_BITS
#define HFB_MAX_JUMP_EXT_BITS 22
#endif
constexpr uint32_t kMaxJumpExtBits = HFB_MAX_JUMP_EXT_BITS;
HFB_HD uint32_t jump_slot(uint32_t key32, uint32_t bits) { return filter2_hash(key32) >> (32 - bits); }
HFB_HD uint32_t jump_slot2(uint32_t key32, uint32_t bits)
{
    return filter2_hash(key32 * 0x9E3779B1u + 0x7F4A7C15u) >> (32 - bits);
}

// Direct-index form for alphabets of at most 4 symbols (filter mode 5: DNA).
// Every pattern has kDnaK..kDnaMaxLen symbols.  The text is packed once per
// scan to 2 bits per byte plus a validity bit per byte (pfac_pack_dna_kernel),
// the first kDnaK symbols of a start are a 16-bit key, and one table blob --
// small enough for shared memory -- answers everything a start needs:
//   bitmap  u32[2048]     bit key: some pattern starts with these 8 symbols
//                         (exact membership, no hashing)
//   wrank   u16[2048]     set bits of the bitmap words before word w
//   first   u16[keys+1]   key rank r -> its patterns [first[r], first[r+1])
//   sym     u64[pats]     pattern symbols, 2 bits each, LSB first
//   meta    u32[pats]     length << 16 | pattern id
// Patterns are sorted by (key, length, id), so a start's records come out in
// (length, id) order.  The blob is built only when the trie accepts exactly
// its dictionary (image.cpp "path ids"): the records of a start are then
// exactly the dictionary patterns that occur there, whatever the trie state.
constexpr uint32_t kDnaK = 8;
constexpr uint32_t kDnaMaxLen = 32;
constexpr uint32_t kDnaMaxPerKey = 32;
constexpr uint32_t kDnaWrankOff = 2048 * 4;          // byte offsets inside the blob
constexpr uint32_t kDnaFirstOff = kDnaWrankOff + 2048 * 2;
HFB_HD uint32_t dna_sym_off(uint32_t keys) { return (kDnaFirstOff + 2 * (keys + 1) + 7) & ~7u; }
HFB_HD uint32_t dna_meta_off(uint32_t keys, uint32_t pats) { return dna_sym_off(keys) + 8 * pats; }
HFB_HD uint32_t dna_blob_bytes(uint32_t keys, uint32_t pats) { return dna_meta_off(keys, pats) + 4 * pats; }
constexpr uint32_t kDnaMaxBlob = 160 * 1024;

// Device view of an uploaded image (plain pointers, passed by value).
struct TrieView {
    const uint32_t* nodes;
    const uint32_t* term_id;   // per node: private pattern id, or kNoId = resolve by key
    const uint32_t* bucket_of; // per node: bucket index or kNoId
    const uint32_t* path_id;   // per node: pattern id naming keyed terminals below it, kNoId, or kKeep
    uint32_t groups;           // grouped format: uint4 records per node
    uint32_t depth_limit;      // 0 = untruncated
    const uint16_t* symtab;    // [256], kNoSym = byte outside the alphabet
    const uint8_t* pat_bytes;
    const uint64_t* pat_off;
    const uint32_t* pat_len;
    const uint64_t* ht_key;
    const uint32_t* ht_id;
    uint64_t ht_mask;
    uint64_t hmul;
    const uint32_t* bk_span;  // uint2 per bucket: {first entry, entry count}
    const uint32_t* bk_entry; // uint4 {pattern id, length, byte offset lo, hi}, sorted by (length, id)
    const uint32_t* filter;
    uint32_t filter_words;
    uint32_t filter_bits; // 0 = filter disabled (every start walks)
    uint32_t filter_k;
    uint32_t pair_shift;  // pair form: 32 - log2(words), i.e. word = (middle * kPairMul) >> pair_shift
    const uint32_t* filter2; // second level, 2^filter2_bits bits
    uint32_t filter2_bits;   // 0 = no second level
    uint32_t sym_bits;       // symbol-key mode (small alphabets): bits per packed symbol (1, 2 or 4),
                             // filter/jump keys are the first filter_k symbols packed LSB-first; 0 = byte keys
    const uint32_t* key4;    // pair pipeline: bitmap over the first 4 bytes of every depth-k path
    uint32_t key4_words;     // (single-probe hash, layout above); 0 = none
    const uint32_t* jump;    // 2^jump_bits uint4 slots
    uint32_t jump_bits;      // 0 = no jump table (walks start at the root)
    const uint32_t* jump_ext; // per slot: first bucket entry + its next 16 pattern bytes, or null
    uint32_t min_emit;
    const uint32_t* filter_l1; // single + L2 form (filter mode 4): the shared-memory level, filter_l1_words
    uint32_t filter_l1_words;  // words (any count: word = umulhi(key * kFilterMul, words), bit key & 31)
    const uint32_t* dna;      // direct-index form (filter mode 5): the table blob (layout above), or null
    uint32_t dna_words;       // blob size in 32-bit words
    uint32_t dna_keys;        // distinct kDnaK-symbol prefixes
    uint32_t dna_pats;        // patterns
    uint32_t dna_symw;        // the alphabet bytes, symbol i in byte i, when symbols follow the
                              // formula ((b >> 1) ^ (b >> 2)) & 3 ("ACGT", "acgt"); else 0
};

// First pattern byte an inline list entry stores (kJumpExtBytes from there):
// byte keys matched bytes [0, k) exactly; packed symbol keys did not (bytes
// outside the alphabet pack as symbol 0), so their compare starts at byte 0.
HFB_HD uint32_t inline_skip(uint32_t filter_k, uint32_t sym_bits) { return sym_bits ? 0u : filter_k & ~3u; }

} // namespace hfb

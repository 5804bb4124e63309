// image.hpp -- host-side builder of the GPU trie image (north-star subsystem
// 1: "the trie compiler still runs on the host but emits a GPU layout").
#pragma once

#include <array>
#include <vector>

#include "../cuda/layout.hpp"
#include "core.hpp"

namespace hfb {

struct GpuImage {
    uint32_t node_count = 0;
    uint32_t groups = 0; // 0 = narrow uint2 records, else uint4 records per node
    std::vector<uint32_t> nodes;
    std::vector<uint32_t> term_id, bucket_of;
    std::vector<uint32_t> path_id; // per node: see image.cpp "path ids" (kKeep on non-unique nodes)
    bool identity = false;
    std::array<uint16_t, 256> symtab{};
    uint32_t depth_limit = 0;

    std::vector<uint8_t> pat_bytes;
    std::vector<uint64_t> pat_off;
    std::vector<uint32_t> pat_len;
    std::vector<uint64_t> ht_key;
    std::vector<uint32_t> ht_id;
    uint64_t ht_mask = 0, hmul = 0;

    std::vector<uint32_t> bk_span, bk_entry; // uint2 / uint4 records, see layout.hpp

    uint32_t filter_k = 0, filter_bits = 0, filter2_bits = 0;
    uint32_t filter_mode = 0; // 0 none, 1 single, 2 pair, 3 packed symbols, 4 single + L2, 5 direct index
    uint32_t sym_bits = 0;    // symbol-key mode: bits per packed symbol (filter_mode 3)
    uint32_t pair_shift = 0;
    double filter_pass = 1.0; // estimated fraction of random starts reaching the walk queue
    uint64_t filter_paths = 0;
    std::vector<uint32_t> filter, filter2;
    std::vector<uint32_t> filter_l1; // filter mode 4: the shared-memory level (kL1Words words)
    std::vector<uint32_t> key4; // pair pipeline: single-probe bitmap over 4-byte path prefixes
    uint32_t jump_bits = 0;     // log2 slots of the depth-k jump table, 0 = none
    std::vector<uint32_t> jump; // uint4 slots, see layout.hpp
    std::vector<uint32_t> jump_ext; // per slot: its inline pattern list (layout.hpp), or empty
    bool dictionary_language = false; // the trie accepts exactly its patterns (image.cpp "path ids")
    std::vector<uint32_t> dna;        // direct-index form (filter_mode 5, layout.hpp), or empty
    uint32_t dna_keys = 0, dna_pats = 0;

    uint32_t min_emit = UINT32_MAX; // shortest depth at which any start can report
    uint64_t reach = 0;             // max bytes one start may read; UINT64_MAX = unbounded
    uint64_t private_terminals = 0, keyed_terminals = 0;

    size_t device_bytes() const;
};

struct ImageOptions {
    uint32_t max_filter_bits = 20; // bitmap of 2^bits bits kept in shared memory (128 KiB)
    uint32_t filter_slack = 6;     // bits above log2(#k-grams): density <= 2^-slack
    uint32_t filter2_slack = 10;   // second level: bits above log2(#k-grams)
    uint32_t max_filter2_bits = 27; // 16 MiB in global memory
    bool jump = true;               // depth-k jump table (HEPFAC_JUMP=0 disables)
    bool jump_ext = true;           // inline pattern lists in the jump table (HEPFAC_JUMP_EXT=0 disables)
    uint32_t filter_mode = 0;       // 0 = cost model, 1 = single, 2 = pair (HEPFAC_FILTER_MODE)
    bool symbol_keys = true;        // packed-symbol filter keys for sigma <= 16 (HEPFAC_SYMBOL_KEYS=0 disables)
    bool dna = true;                // direct-index form for sigma <= 4 (HEPFAC_DNA=0 disables)
};

ImageOptions image_options_from_env();
GpuImage build_gpu_image(const Trie& t, const ImageOptions& opt);

} // namespace hfb

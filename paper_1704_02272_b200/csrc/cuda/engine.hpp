// engine.hpp -- host interface of the GPU match engine (csrc/cuda/engine.cu).
// Used by the C ABI layer (csrc/host/capi.cpp); nothing here exposes CUDA types.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "../host/core.hpp"

namespace hfb {

// Host-side result of a scan: the reference's vector<MatchResult>
// (capi.cpp:31-33), held as a flat array of hepfac_match_t.
// Lists of 1 MiB or more sit in pinned (page-locked) host memory from a
// process-wide pool, so their D2H runs at PCIe speed; destroy returns the
// block to the pool.
struct MatchList {
    hepfac_match_t* data = nullptr;
    size_t size = 0;
    size_t cap = 0;      // records the block holds
    bool pinned = false;
    MatchList() = default;
    MatchList(const MatchList&) = delete;
    ~MatchList();
    void allocate(size_t n);  // size = n, contents undefined
    void reserve(size_t n);   // capacity >= n, keeps the first `size` records
    void release();
};

// Timing breakdown of the most recent hepfac_scan on this thread (device
// events on the engine's stream).
struct ScanStats {
    double h2d_ms = 0, kernel_ms = 0, d2h_ms = 0, total_ms = 0;
    uint64_t bytes = 0, matches = 0;
    uint32_t kernel_launches = 0, chunks = 0, relaunches = 0;
    int device = -1;
    bool staged = false; // pageable text went through the pinned staging ring
};

// hepfac_scan: every occurrence, sorted by (start, length, id).
std::unique_ptr<MatchList> gpu_scan(const Trie& t, const uint8_t* host_text, uint64_t bytes);

// Shard scan: `text` holds global bytes [g0, g0 + avail); report starts in
// [g0, g0 + owned).  Walks stop at g0 + avail, which the caller sets to
// min(N, g0 + owned + halo) so results equal the full-text scan's.
std::unique_ptr<MatchList> gpu_scan_shard(const Trie& t, const uint8_t* host_text, uint64_t avail,
                                          uint64_t owned, uint64_t g0);

// Bytes of right context a shard needs (reach - 1); UINT64_MAX if unbounded.
uint64_t gpu_halo(const Trie& t);

// hepfac_run_throughput (reference bench.cpp:52-78): 1 warm-up + `runs` timed
// scans of device-resident text.  seconds = mean kernel time, merge_seconds =
// mean time to hand the sorted list back to the host.
struct Throughput {
    double seconds = 0, merge_seconds = 0;
    uint64_t matches = 0;
};
Throughput gpu_run_throughput(const Trie& t, const uint8_t* host_text, uint64_t bytes, uint32_t runs);

const ScanStats& last_scan_stats();

// Device-resident benchmark session (hepfac_b200.h).
struct Session;
Session* session_create(const Trie& t, const uint8_t* host_text, uint64_t bytes, uint64_t offset, uint64_t owned);
void session_run(Session* s, uint32_t iterations, int flush_l2, double* ms_each);
uint64_t session_matches(Session* s);
// Per-kernel device times of the last run: first = filter pass (or the fused
// scan kernel), second = candidate-walking pass (0 without the pair pipeline).
void session_split(Session* s, uint32_t n, double* first_ms, double* second_ms, uint32_t* kernels_per_scan);
std::unique_ptr<MatchList> session_fetch(Session* s);
void session_destroy(Session* s);

struct LayoutInfo {
    uint32_t node_count, groups, record_bytes, filter_k, filter_bits, min_emit, smem_bytes,
        blocks_per_sm, sm_count, identity;
    uint64_t filter_paths, reach, device_bytes, private_terminals, keyed_terminals;
    uint32_t filter_mode, filter_pass_ppm, filter2_bits;
};
LayoutInfo layout_info(const Trie& t);

int device_count();

// Frees every pooled workspace (device buffers, streams) and pinned block
// that no call is using (hepfac_b200_trim).
void trim_pools();

} // namespace hfb

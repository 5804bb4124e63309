/*
 * hepfac_b200.h -- additive, GPU-specific entry points of libhepfac (B200).
 *
 * Nothing here is needed by a program written against the reference
 * hepfac.h; these calls expose what only a GPU engine has: shard scans for
 * multi-GPU / multi-process callers, device-resident benchmarking, the
 * device-timed breakdown of the last hepfac_scan, and the GPU trie image.
 */
#ifndef HEPFAC_B200_H
#define HEPFAC_B200_H

#include "hepfac.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Number of visible CUDA devices (0 when none). */
int hepfac_b200_device_count(void);

/* Bytes of right context a shard needs so that its starts see the same walks
 * as a whole-text scan: (longest walk - 1).  UINT64_MAX when unbounded (a
 * cyclic loaded trie), in which case shards cannot be used. */
hepfac_status_t hepfac_b200_halo(const hepfac_trie_t* trie, uint64_t* halo);

/* Shard scan.  `text` holds the global bytes [offset, offset + bytes); the
 * shard reports starts [offset, offset + owned) with GLOBAL start positions.
 * Walks stop at offset + bytes, so pass bytes = min(N - offset, owned + halo)
 * to reproduce the full-text result for those starts. */
hepfac_status_t hepfac_b200_scan_shard(const hepfac_trie_t* trie, const uint8_t* text,
                                       uint64_t bytes, uint64_t offset, uint64_t owned,
                                       hepfac_match_list_t** out);

/* Device-timed breakdown of the calling thread's most recent hepfac_scan /
 * hepfac_b200_scan_shard (CUDA events on the engine's stream). */
typedef struct hepfac_b200_scan_stats {
    double h2d_ms;
    double kernel_ms;
    double d2h_ms;
    double total_ms;
    uint64_t bytes;
    uint64_t matches;
    uint32_t kernel_launches;
    uint32_t chunks;
    uint32_t relaunches;
    int32_t device;
    uint32_t staged;   /* 1: the text was pageable and went through the pinned staging ring */
} hepfac_b200_scan_stats_t;

hepfac_status_t hepfac_b200_last_scan_stats(hepfac_b200_scan_stats_t* out);

/* Frees every pooled per-call workspace (device buffers, streams) and pooled
 * pinned host block that no call is using.  Calls after it re-allocate on
 * demand.  Pooled workspaces otherwise keep at most HEPFAC_POOL_KEEP_MIB
 * (default 2048) MiB of device buffers each between calls. */
hepfac_status_t hepfac_b200_trim(void);

/* Device-resident session: text uploaded once, scanned repeatedly.  Same
 * shard convention as hepfac_b200_scan_shard (offset = 0, owned = bytes for a
 * whole text). */
typedef struct hepfac_b200_session hepfac_b200_session_t;
hepfac_status_t hepfac_b200_session_create(const hepfac_trie_t* trie, const uint8_t* text,
                                           uint64_t bytes, uint64_t offset, uint64_t owned,
                                           hepfac_b200_session_t** out);
/* Runs `iterations` scans; ms_each[i] (may be NULL) = device time of scan i.
 * flush_l2 != 0 evicts L2 before each (untimed). */
hepfac_status_t hepfac_b200_session_run(hepfac_b200_session_t* session, uint32_t iterations,
                                        int flush_l2, double* ms_each, uint64_t* matches);
/* Per-kernel device times of the last run's scans (CUDA events on the
 * engine's stream): first = the filter pass of the pair pipeline, or the fused
 * scan kernel; second = the candidate-walking pass (0 when there is none).
 * *kernels_per_scan (may be NULL) = kernel launches per scan: 1 (fused), 2
 * (filter + walking pass) or 3 (symbol packing + filter + walking pass; the
 * packing pass is timed with the filter pass). */
hepfac_status_t hepfac_b200_session_kernel_ms(hepfac_b200_session_t* session, uint32_t iterations,
                                              double* first_ms, double* second_ms, uint32_t* kernels_per_scan);
/* Copies the last run's sorted matches to the host. */
hepfac_status_t hepfac_b200_session_fetch(hepfac_b200_session_t* session,
                                          hepfac_match_list_t** out);
void hepfac_b200_session_destroy(hepfac_b200_session_t* session);

/* GPU trie image of a trie on the current device. */
typedef struct hepfac_b200_layout_info {
    uint32_t node_count;
    uint32_t groups;       /* 0 = 8-byte narrow records, else 16-byte records per node */
    uint32_t record_bytes; /* bytes per node in the GPU image */
    uint32_t filter_k;     /* bytes hashed by the start filter */
    uint32_t filter_bits;  /* log2 filter bitmap bits; 0 = filter disabled */
    uint32_t min_emit;     /* shortest report depth; UINT32_MAX = nothing can match */
    uint32_t smem_bytes;
    uint32_t blocks_per_sm;
    uint32_t sm_count;
    uint32_t identity;     /* byte == symbol */
    uint64_t filter_paths; /* distinct depth-k path strings */
    uint64_t reach;        /* longest byte span of one start */
    uint64_t device_bytes;
    uint64_t private_terminals;
    uint64_t keyed_terminals;
    uint32_t filter_mode;     /* 0 none, 1 single probe per start, 2 pair probes (one per two starts),
                                 3 packed-symbol keys, 4 single probe + L2-resident bitmap (two-pass) */
    uint32_t filter_pass_ppm; /* estimated random starts per million that reach the walk queue */
    uint32_t filter2_bits;    /* log2 bits of the L2-resident filter level; 0 = none */
} hepfac_b200_layout_info_t;

hepfac_status_t hepfac_b200_layout_info(const hepfac_trie_t* trie, hepfac_b200_layout_info_t* out);

#ifdef __cplusplus
}
#endif

#endif /* HEPFAC_B200_H */

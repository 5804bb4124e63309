/*
 * pfac_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's CPU match path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.
 * Nothing in paper_1704_02272_b200/ links, loads or calls this code.
 *
 * Parity pinning: tests/test_oracle.py checks both restatements against the
 * reference's golden vectors (test_capi.cpp:81-96, test_scan.cpp:19-41,90-101)
 * and against the unmodified reference library compiled from its sources into
 * oracle/_ref/ (oracle/Makefile).
 */
#ifndef PFAC_ORACLE_H
#define PFAC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same 16-byte record as hepfac_match_t (hepfac.h:137-141). */
typedef struct oracle_match {
    uint64_t start;
    uint32_t length;
    uint32_t pattern_id;
} oracle_match_t;

/* Brute force: every pattern at every offset, memcmp, then sort by
 * (start, length, id).  Restates naive_search.hpp:17-31.
 * Returns the total number of matches; writes min(total, cap) records. */
uint64_t oracle_naive_find_all(const uint8_t* text, uint64_t n, const uint8_t* pattern_bytes,
                               const uint64_t* pattern_offsets, const uint32_t* pattern_lengths,
                               uint32_t pattern_count, oracle_match_t* out, uint64_t cap);

/* Trie description in the reference's canonical cell layout
 * (trie.hpp:45-59): node i = cells[i*(words+1) .. +words] bitmap words, then
 * the offset word (MSB = terminal).  Buckets are given as a CSR over the
 * sorted list of bucket nodes (trie.hpp:116-120). */
typedef struct oracle_trie {
    const uint32_t* cells;
    uint32_t node_count;
    uint32_t words;
    const int16_t* symbol_of; /* [256], -1 = byte not in the alphabet */
    uint32_t depth_limit;     /* 0 = not truncated */
    const uint8_t* pattern_bytes;
    const uint64_t* pattern_offsets;
    const uint32_t* pattern_lengths;
    uint32_t pattern_count;
    const uint32_t* bucket_nodes;   /* ascending */
    const uint32_t* bucket_starts;  /* bucket_count + 1 entries */
    const uint32_t* bucket_ids;     /* ascending within each bucket */
    uint32_t bucket_count;
} oracle_trie_t;

/* Failure-less walk from every offset (scan.cpp:69-119 with the walk of
 * scan.cpp:20-51, transition of trie.hpp:68-79, id lookup of trie.hpp:103-107,
 * bucket verification of scan.cpp:37-49), merged and sorted like
 * scan.cpp:104-111.  Returns the total count, or UINT64_MAX when a terminal
 * spells no dictionary pattern (the reference's logic_error, scan.cpp:34). */
uint64_t oracle_walk_scan(const oracle_trie_t* trie, const uint8_t* text, uint64_t n,
                          oracle_match_t* out, uint64_t cap);

/* Single transition (trie.hpp:68-79); UINT32_MAX on a miss. */
uint32_t oracle_transition(const oracle_trie_t* trie, uint32_t node, uint8_t byte);

#ifdef __cplusplus
}
#endif

#endif

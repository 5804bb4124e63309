/*
 * pfac_oracle.c -- TEST INFRASTRUCTURE ONLY (see pfac_oracle.h).
 *
 * A deliberately simple, scalar C restatement of the reference's match path.
 * It is the checker the CUDA path is compared against; it is never the thing
 * measured for `value`/`e2e` and never linked into the product library.
 */
#include "pfac_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---- growable output ---------------------------------------------------- */

typedef struct vec {
    oracle_match_t* data;
    uint64_t size, cap;
    int oom;
} vec_t;

static void vec_push(vec_t* v, uint64_t start, uint32_t len, uint32_t id)
{
    if (v->oom) return;
    if (v->size == v->cap) {
        uint64_t nc = v->cap ? v->cap * 2 : 1024;
        oracle_match_t* nd = (oracle_match_t*)realloc(v->data, nc * sizeof(oracle_match_t));
        if (!nd) {
            v->oom = 1;
            return;
        }
        v->data = nd;
        v->cap = nc;
    }
    v->data[v->size].start = start;
    v->data[v->size].length = len;
    v->data[v->size].pattern_id = id;
    v->size++;
}

/* Order of MatchResult::operator<=> (scan.hpp:17-23). */
static int cmp_match(const void* pa, const void* pb)
{
    const oracle_match_t* a = (const oracle_match_t*)pa;
    const oracle_match_t* b = (const oracle_match_t*)pb;
    if (a->start != b->start) return a->start < b->start ? -1 : 1;
    if (a->length != b->length) return a->length < b->length ? -1 : 1;
    if (a->pattern_id != b->pattern_id) return a->pattern_id < b->pattern_id ? -1 : 1;
    return 0;
}

static uint64_t finish(vec_t* v, oracle_match_t* out, uint64_t cap)
{
    if (v->oom) {
        free(v->data);
        return UINT64_MAX - 1;
    }
    qsort(v->data, (size_t)v->size, sizeof(oracle_match_t), cmp_match);
    uint64_t k = v->size < cap ? v->size : cap;
    if (k && out) memcpy(out, v->data, (size_t)k * sizeof(oracle_match_t));
    free(v->data);
    return v->size;
}

/* ---- naive_find_all: naive_search.hpp:17-31 ----------------------------- */

uint64_t oracle_naive_find_all(const uint8_t* text, uint64_t n, const uint8_t* pattern_bytes,
                               const uint64_t* pattern_offsets, const uint32_t* pattern_lengths,
                               uint32_t pattern_count, oracle_match_t* out, uint64_t cap)
{
    vec_t v = {0};
    for (uint64_t start = 0; start < n; ++start) {            /* naive_search.hpp:21 */
        for (uint32_t id = 0; id < pattern_count; ++id) {      /* :22 */
            uint32_t len = pattern_lengths[id];
            if (start + len > n) continue;                     /* :24 */
            const uint8_t* p = pattern_bytes + pattern_offsets[id];
            if (text[start] != p[0]) continue; /* cheap pre-check, same predicate */
            if (memcmp(text + start, p, len) == 0) vec_push(&v, start, len, id); /* :25-26 */
        }
    }
    return finish(&v, out, cap);                               /* sort :29 */
}

/* ---- dictionary: trie.hpp:103-107 (hash of the matched slice) ----------- */

typedef struct dict {
    uint32_t* slots; /* id + 1, 0 = empty */
    uint64_t mask;
} dict_t;

static uint64_t fnv1a(const uint8_t* s, uint32_t len)
{
    uint64_t h = 1469598103934665603ull;
    for (uint32_t i = 0; i < len; ++i) {
        h ^= s[i];
        h *= 1099511628211ull;
    }
    return h ^ len;
}

static int dict_build(dict_t* d, const oracle_trie_t* t)
{
    uint64_t cap = 16;
    while (cap < 2ull * t->pattern_count + 16) cap <<= 1;
    d->slots = (uint32_t*)calloc((size_t)cap, sizeof(uint32_t));
    if (!d->slots) return 0;
    d->mask = cap - 1;
    for (uint32_t id = 0; id < t->pattern_count; ++id) {
        const uint8_t* p = t->pattern_bytes + t->pattern_offsets[id];
        uint64_t h = fnv1a(p, t->pattern_lengths[id]) & d->mask;
        while (d->slots[h]) h = (h + 1) & d->mask;
        d->slots[h] = id + 1;
    }
    return 1;
}

static int64_t dict_find(const dict_t* d, const oracle_trie_t* t, const uint8_t* s, uint32_t len)
{
    uint64_t h = fnv1a(s, len) & d->mask;
    while (d->slots[h]) {
        uint32_t id = d->slots[h] - 1;
        if (t->pattern_lengths[id] == len &&
            memcmp(t->pattern_bytes + t->pattern_offsets[id], s, len) == 0)
            return id;
        h = (h + 1) & d->mask;
    }
    return -1;
}

/* ---- transition: trie.hpp:68-79 ---------------------------------------- */

uint32_t oracle_transition(const oracle_trie_t* t, uint32_t node, uint8_t byte)
{
    int sym = t->symbol_of[byte];                              /* trie.hpp:70 */
    if (sym < 0) return UINT32_MAX;                            /* :71 */
    const uint32_t* c = t->cells + (uint64_t)node * (t->words + 1);
    unsigned w = (unsigned)sym >> 5, b = (unsigned)sym & 31u;  /* :73-74 */
    if (!((c[w] >> b) & 1u)) return UINT32_MAX;               /* :75 */
    uint32_t rank = (uint32_t)__builtin_popcount(c[w] & ((1u << b) - 1u)); /* :76 */
    for (unsigned i = 0; i < w; ++i) rank += (uint32_t)__builtin_popcount(c[i]); /* :77 */
    return (c[t->words] & 0x7FFFFFFFu) + rank;                /* :78 */
}

static int terminal(const oracle_trie_t* t, uint32_t node)
{
    return (t->cells[(uint64_t)node * (t->words + 1) + t->words] & 0x80000000u) != 0; /* trie.hpp:81 */
}

static int64_t bucket_index(const oracle_trie_t* t, uint32_t node)
{
    uint32_t lo = 0, hi = t->bucket_count;
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (t->bucket_nodes[mid] < node) lo = mid + 1;
        else hi = mid;
    }
    if (lo < t->bucket_count && t->bucket_nodes[lo] == node) return lo;
    return -1;
}

/* ---- walk: scan.cpp:20-51 ---------------------------------------------- */

static int walk(const oracle_trie_t* t, const dict_t* d, const uint8_t* text, uint64_t n,
                uint64_t start, vec_t* out)
{
    uint32_t node = 0;
    uint64_t pos = start;
    const uint64_t limit = t->depth_limit;                    /* scan.cpp:25 */
    while (pos < n) {                                          /* :26 */
        node = oracle_transition(t, node, text[pos]);          /* :27 */
        if (node == UINT32_MAX) return 1;                      /* :28 */
        ++pos;
        if (terminal(t, node)) {                               /* :30 */
            uint32_t len = (uint32_t)(pos - start);
            int64_t id = dict_find(d, t, text + start, len);   /* :32-33 */
            if (id < 0) return 0;                              /* :34 logic_error */
            vec_push(out, start, len, (uint32_t)id);           /* :35 */
        }
        if (pos - start == limit) {                            /* :39 */
            int64_t b = bucket_index(t, node);                 /* :40 */
            if (b >= 0) {
                for (uint32_t k = t->bucket_starts[b]; k < t->bucket_starts[b + 1]; ++k) {
                    uint32_t id = t->bucket_ids[k];            /* :41 */
                    uint32_t plen = t->pattern_lengths[id];
                    if (start + plen > n) continue;            /* :43 */
                    if (memcmp(text + start, t->pattern_bytes + t->pattern_offsets[id], plen) == 0)
                        vec_push(out, start, plen, id);        /* :44-45 */
                }
            }
            return 1;                                          /* :48 */
        }
    }
    return 1;
}

/* ---- scan: scan.cpp:69-119 (one worker; output is worker-invariant) ----- */

uint64_t oracle_walk_scan(const oracle_trie_t* t, const uint8_t* text, uint64_t n,
                          oracle_match_t* out, uint64_t cap)
{
    dict_t d;
    if (!dict_build(&d, t)) return UINT64_MAX - 1;
    vec_t v = {0};
    for (uint64_t start = 0; start < n; ++start) {             /* scan.cpp:86 */
        if (!walk(t, &d, text, n, start, &v)) {
            free(d.slots);
            free(v.data);
            return UINT64_MAX;
        }
    }
    free(d.slots);
    return finish(&v, out, cap);                               /* scan.cpp:111 */
}

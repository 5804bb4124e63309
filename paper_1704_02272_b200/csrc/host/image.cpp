// image.cpp -- canonical trie -> GPU image.
//
// What the kernel needs that the canonical cells do not give directly:
//   * one-load transitions (grouped records with per-group rank bases);
//   * pattern ids at terminals.  The reference hashes the matched slice into
//     its dictionary (trie.hpp:103-107) because stage-1/2 terminals are shared
//     (SPEC.md:368).  Here every terminal reached by exactly one root path gets
//     its id baked in; shared terminals resolve by a 64-bit slice key into an
//     open-addressing table, followed by a byte compare;
//   * verification buckets as a CSR sorted by (length, id), so a start's
//     matches come out already in (length, id) order (scan.hpp:17-23);
//   * the start filter: every start that can report passes through a node at
//     depth k = min(8, shortest report depth), so the set of depth-k path
//     strings, hashed into a bitmap, rejects most starts with one shared-memory
//     probe;
//   * reach, the longest byte span one start can read (the halo of a shard).
#include "image.hpp"

#include <algorithm>
#include <atomic>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

namespace hfb {

size_t GpuImage::device_bytes() const
{
    return nodes.size() * 4 + term_id.size() * 4 + bucket_of.size() * 4 + pat_bytes.size() +
           pat_off.size() * 8 + pat_len.size() * 4 + ht_key.size() * 8 + ht_id.size() * 4 +
           bk_span.size() * 4 + bk_entry.size() * 4 + path_id.size() * 4 + filter.size() * 4 + filter2.size() * 4 + key4.size() * 4 + jump.size() * 4 + jump_ext.size() * 4 + dna.size() * 4 + filter_l1.size() * 4 + 512;
}

ImageOptions image_options_from_env()
{
    ImageOptions o;
    if (const char* s = std::getenv("HEPFAC_JUMP")) o.jump = std::strtol(s, nullptr, 10) != 0;
    if (const char* s = std::getenv("HEPFAC_JUMP_EXT")) o.jump_ext = std::strtol(s, nullptr, 10) != 0;
    if (const char* s = std::getenv("HEPFAC_SYMBOL_KEYS")) o.symbol_keys = std::strtol(s, nullptr, 10) != 0;
    if (const char* s = std::getenv("HEPFAC_DNA")) o.dna = std::strtol(s, nullptr, 10) != 0;
    if (const char* s = std::getenv("HEPFAC_FILTER_MODE")) {
        const std::string m = s;
        o.filter_mode = m == "single" ? 1u : (m == "pair" ? 2u : (m == "l2" ? 4u : 0u));
    }
    return o;
}

namespace {

uint32_t ceil_log2(uint64_t x)
{
    uint32_t b = 0;
    while ((uint64_t(1) << b) < x) ++b;
    return b;
}

// Cuckoo jump table (layout.hpp): entries are 8-word slots whose words 0/1
// are the key; a slot with word 2 == kNoId is empty.  Grows until every key
// places (load <= 1/2 to start).  `lists[i]` (optional) names every pattern
// with entry i's k-prefix when there are at most kJumpExtEntries of them
// (flags bit 2, see inline_lists); up to 2^kMaxJumpExtBits slots those go to
// the slot's extension (layout.hpp), otherwise bit 2 is cleared.
using JumpEntry = std::array<uint32_t, kJumpWords>;
using InlineList = std::array<uint32_t, kJumpExtEntries>;

void build_jump_table(GpuImage& im, const std::vector<JumpEntry>& entries, const std::vector<InlineList>& lists)
{
    constexpr size_t W = kJumpWords;
    uint32_t jb = std::max<uint32_t>(ceil_log2(entries.size()) + 1, 4);
    for (;; ++jb) {
        const size_t slots = size_t(1) << jb;
        std::vector<uint32_t> tab(W * slots, 0u);
        std::vector<uint32_t> where(slots, kNoId); // slot -> entry index
        for (size_t s = 0; s < slots; ++s) tab[W * s + 2] = kNoId;
        bool ok = true;
        for (size_t i = 0; i < entries.size() && ok; ++i) {
            JumpEntry cur = entries[i];
            uint32_t ci = uint32_t(i);
            uint32_t pos = jump_slot(cur[0] ^ (cur[1] * 0x85EBCA77u), jb);
            for (int kick = 0;; ++kick) {
                if (kick > 500) {
                    ok = false;
                    break;
                }
                uint32_t* slot = &tab[W * pos];
                if (slot[2] == kNoId) {
                    std::copy(cur.begin(), cur.end(), slot);
                    where[pos] = ci;
                    break;
                }
                const uint32_t k32 = cur[0] ^ (cur[1] * 0x85EBCA77u);
                const uint32_t alt = pos == jump_slot(k32, jb) ? jump_slot2(k32, jb) : jump_slot(k32, jb);
                uint32_t* other = &tab[W * alt];
                if (other[2] == kNoId) {
                    std::copy(cur.begin(), cur.end(), other);
                    where[alt] = ci;
                    break;
                }
                // evict the occupant of `pos` and move it to its other slot
                JumpEntry ev;
                std::copy(slot, slot + W, ev.begin());
                const uint32_t ei = where[pos];
                std::copy(cur.begin(), cur.end(), slot);
                where[pos] = ci;
                cur = ev;
                ci = ei;
                const uint32_t ek = cur[0] ^ (cur[1] * 0x85EBCA77u);
                pos = pos == jump_slot(ek, jb) ? jump_slot2(ek, jb) : jump_slot(ek, jb);
            }
        }
        if (ok) {
            im.jump_bits = jb;
            im.jump = std::move(tab);
            im.jump_ext.clear();
            if (!lists.empty() && jb <= kMaxJumpExtBits) {
                const uint32_t skip = inline_skip(im.filter_k, im.sym_bits);
                im.jump_ext.assign(kJumpExtWords * slots, 0u);
                for (size_t s = 0; s < slots; ++s) {
                    if (where[s] == kNoId || !(im.jump[W * s + 6] & kJumpInline)) continue;
                    const InlineList& l = lists[where[s]];
                    for (uint32_t j = 0; j < kJumpExtEntries && l[j] != kNoId; ++j) {
                        uint32_t* x = &im.jump_ext[kJumpExtWords * s + kJumpExtEntryWords * j];
                        const uint32_t id = l[j], len = im.pat_len[id];
                        x[0] = id;
                        x[1] = len;
                        for (uint32_t b = skip; b < std::min(len, skip + kJumpExtBytes); ++b)
                            x[2 + (b - skip) / 4] |= uint32_t(im.pat_bytes[im.pat_off[id] + b]) << (8 * ((b - skip) & 3));
                    }
                }
            } else {
                for (size_t s = 0; s < slots; ++s) im.jump[W * s + 6] &= ~(kJumpInline | (3u << kJumpInlineShift));
            }
            return;
        }
        if (jb > 30) fail(HEPFAC_ERR_NOMEM, "cannot place the jump table");
    }
}

// Every pattern whose first k bytes (sb == 0) or k packed symbols (sb bits
// each) give jump key keys[i], sorted by (length, id), when there are at most
// kJumpExtEntries of them; kNoId-filled otherwise.  For a trie that accepts
// exactly its dictionary (image.cpp "path ids") these are all the records a
// start reaching that key can emit, truncated or not, so the walk reduces to
// verifying them.  Sets flags bit 2 and the count on the entries it fills.
std::vector<InlineList> inline_lists(const Trie& t, const GpuImage& im, std::vector<JumpEntry>& entries,
                                     const std::vector<uint64_t>& keys, uint32_t k, uint32_t sb)
{
    const size_t K = keys.size(), P = t.patterns.size();
    // the keys sorted (each once: the trie spells a string by one path), for
    // binary-search lookups from all host threads
    std::vector<std::pair<uint64_t, uint32_t>> sorted(K);
    for (size_t i = 0; i < K; ++i) sorted[i] = {keys[i], uint32_t(i)};
    std::sort(sorted.begin(), sorted.end());
    std::vector<uint32_t> key_of(P);
    std::atomic<bool> off{false};
    parallel_slices(P, 4096, [&](size_t b, size_t e) {
        for (size_t id = b; id < e; ++id) {
            const auto& p = t.patterns[id];
            if (p.size() < k) { // cannot happen when k <= min_emit; stay on the walk
                off = true;
                return;
            }
            uint64_t key = 0;
            for (uint32_t i = 0; i < k; ++i) {
                const uint8_t c = uint8_t(p[i]);
                key |= sb ? uint64_t(uint32_t(t.alphabet.symbol_of(c))) << (sb * i) : uint64_t(c) << (8 * i);
            }
            const auto it = std::lower_bound(sorted.begin(), sorted.end(), std::make_pair(key, 0u));
            if (it == sorted.end() || it->first != key) { // a pattern off the trie: not its dictionary
                off = true;
                return;
            }
            key_of[id] = it->second;
        }
    });
    if (off) return {};
    // every key's patterns in id order (counting sort)
    std::vector<uint32_t> first(K + 1, 0);
    for (size_t id = 0; id < P; ++id) ++first[key_of[id] + 1];
    for (size_t i = 0; i < K; ++i) first[i + 1] += first[i];
    std::vector<uint32_t> flat(P), next(first.begin(), first.end() - 1);
    for (size_t id = 0; id < P; ++id) flat[next[key_of[id]]++] = uint32_t(id);
    std::vector<InlineList> lists(K);
    parallel_slices(K, 1 << 14, [&](size_t b, size_t e) {
        for (size_t i = b; i < e; ++i) {
            lists[i].fill(kNoId);
            const uint32_t n = first[i + 1] - first[i];
            if (n == 0 || n > kJumpExtEntries) continue;
            uint32_t* v = flat.data() + first[i];
            std::sort(v, v + n, [&](uint32_t x, uint32_t y) {
                return im.pat_len[x] != im.pat_len[y] ? im.pat_len[x] < im.pat_len[y] : x < y;
            });
            std::copy(v, v + n, lists[i].begin());
            entries[i][6] |= kJumpInline | (n << kJumpInlineShift);
        }
    });
    return lists;
}

} // namespace

GpuImage build_gpu_image(const Trie& t, const ImageOptions& opt)
{
    GpuImage im;
    const uint32_t n = t.node_count;
    if (n >= kMaxGpuNodes) fail(HEPFAC_ERR_NOMEM, "trie too large for the GPU image (>= 2^30 nodes)");
    im.node_count = n;

    // Structural validation: a loaded .htri is only checked for offset < n by
    // the format (reference trie_io.cpp:155-159); child runs must fit too.
    std::vector<uint32_t> kids(n);
    std::atomic<bool> past{false};
    parallel_slices(n, 1 << 16, [&](size_t b, size_t e) {
        for (size_t u = b; u < e; ++u) {
            kids[u] = t.child_count(uint32_t(u));
            if (kids[u] && uint64_t(t.offset(uint32_t(u))) + kids[u] > n) past = true;
        }
    });
    if (past) fail(HEPFAC_ERR_FORMAT, "trie file offset out of range (child run past the node array)");

    // ---- alphabet --------------------------------------------------------
    im.identity = t.alphabet.is_identity();
    for (unsigned b = 0; b < 256; ++b) {
        int s = t.alphabet.symbol_of(uint8_t(b));
        im.symtab[b] = s < 0 ? kNoSym : uint16_t(s);
    }
    im.depth_limit = t.depth_limit.value_or(0);

    // ---- dictionary + slice-key table -------------------------------------
    const size_t P = t.patterns.size();
    im.pat_off.resize(P);
    im.pat_len.resize(P);
    for (size_t i = 0; i < P; ++i) {
        im.pat_off[i] = im.pat_bytes.size(); // 4-byte aligned, zero padded: word compares
        im.pat_len[i] = uint32_t(t.patterns[i].size());
        im.pat_bytes.insert(im.pat_bytes.end(), t.patterns[i].begin(), t.patterns[i].end());
        im.pat_bytes.resize((im.pat_bytes.size() + 3) & ~size_t(3), 0);
    }
    im.pat_bytes.resize(im.pat_bytes.size() + 8, 0); // word reads may overrun the last pattern
    std::vector<uint64_t> keys(P);
    for (uint64_t attempt = 0;; ++attempt) {
        im.hmul = 0x100000001B3ull + 2 * attempt * 0x9E3779B97F4A7C15ull; // odd multipliers
        parallel_slices(P, 4096, [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) {
                const std::string& p = t.patterns[i];
                uint64_t h = 0;
                for (size_t o = 0; o < p.size(); o += 4) {
                    uint32_t w = 0;
                    for (size_t c = 0; c < 4 && o + c < p.size(); ++c) w |= uint32_t(uint8_t(p[o + c])) << (8 * c);
                    h = slice_step(h, im.hmul, w);
                }
                keys[i] = slice_key(h, uint32_t(p.size()));
            }
        });
        std::vector<uint64_t> sorted(keys);
        std::sort(sorted.begin(), sorted.end());
        if (std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end()) break;
        if (attempt > 64) fail(HEPFAC_ERR_INTERNAL, "cannot find collision-free slice keys");
    }
    const uint64_t slots = uint64_t(1) << std::max<uint32_t>(4, ceil_log2(2 * P + 1));
    im.ht_mask = slots - 1;
    im.ht_key.assign(slots, 0);
    im.ht_id.assign(slots, kNoId);
    for (size_t i = 0; i < P; ++i) {
        uint64_t s = mix64(keys[i]) & im.ht_mask;
        while (im.ht_id[s] != kNoId) s = (s + 1) & im.ht_mask;
        im.ht_key[s] = keys[i];
        im.ht_id[s] = uint32_t(i);
    }

    // ---- terminal ids: baked in where the node spells exactly one string ----
    std::vector<uint32_t> indeg(n, 0);
    parallel_slices(n, 1 << 16, [&](size_t b, size_t e) {
        for (size_t u = b; u < e; ++u)
            for (uint32_t i = 0; i < kids[u]; ++i)
                std::atomic_ref<uint32_t>(indeg[t.offset(uint32_t(u)) + i]).fetch_add(1, std::memory_order_relaxed);
    });
    std::vector<uint8_t> unique_path(n, 0);
    {
        std::vector<uint32_t> q{0};
        unique_path[0] = indeg[0] == 0;
        for (size_t h = 0; h < q.size() && unique_path[0]; ++h) {
            const uint32_t u = q[h];
            for (uint32_t i = 0; i < kids[u]; ++i) {
                const uint32_t c = t.offset(u) + i;
                if (indeg[c] == 1 && !unique_path[c]) {
                    unique_path[c] = 1;
                    q.push_back(c);
                }
            }
        }
    }
    im.term_id.assign(n, kNoId);
    // every pattern's walk, in parallel: a node on a unique path spells one
    // string, so no two patterns write the same entry
    parallel_slices(P, 4096, [&](size_t b, size_t e) {
        for (size_t id = b; id < e; ++id) {
            uint32_t node = 0;
            for (unsigned char c : t.patterns[id]) {
                node = t.transition(node, c);
                if (node >= n) break;
            }
            if (node < n && node != 0 && t.terminal(node) && unique_path[node]) im.term_id[node] = uint32_t(id);
        }
    });

    // ---- path ids: keyed terminals named by the walk's path ------------------
    // A pattern whose terminal is shared (keyed) is still determined by the
    // deepest path-unique node U on its path when U leads to no other keyed
    // terminal and no terminal lies between U and the end.  path_id[U] = that
    // pattern (kNoId if U is ambiguous); path_id of a non-unique node = kKeep.
    // The walk carries the last path_id it met and names a keyed terminal with
    // it; only kNoId falls back to the slice-key lookup.
    // They are only sound when the trie accepts exactly its dictionary (true
    // for every trie this library builds or compresses; a hand-made .htri may
    // carry terminals that spell no pattern, which must keep failing like the
    // reference).  Check: the number of root-to-terminal paths (Kahn order over
    // the DAG; a cycle disables path ids) equals the number of patterns whose
    // full path ends at a terminal.
    bool dictionary_language = true;
    std::vector<uint32_t> order; // Kahn (topological) order of the DAG, when it is one
    {
        std::vector<uint32_t> deg = indeg;
        order.reserve(n);
        if (deg[0] != 0) dictionary_language = false;
        else order.push_back(0);
        for (size_t h = 0; h < order.size(); ++h) {
            const uint32_t u = order[h];
            for (uint32_t i = 0; i < kids[u]; ++i)
                if (--deg[t.offset(u) + i] == 0) order.push_back(t.offset(u) + i);
        }
        std::vector<uint64_t> paths(n, 0);
        uint64_t terminal_paths = 0;
        constexpr uint64_t kCap = uint64_t(1) << 62;
        if (dictionary_language) {
            paths[0] = 1;
            for (uint32_t u : order) {
                if (u != 0 && t.terminal(u)) terminal_paths = std::min(kCap, terminal_paths + paths[u]);
                for (uint32_t i = 0; i < kids[u]; ++i) {
                    uint64_t& c = paths[t.offset(u) + i];
                    c = std::min(kCap, c + paths[u]);
                }
            }
        }
        std::atomic<uint64_t> spelled{0};
        if (dictionary_language)
            parallel_slices(P, 4096, [&](size_t b, size_t e) {
                uint64_t k = 0;
                for (size_t id = b; id < e; ++id) {
                    uint32_t node = 0;
                    bool full = true;
                    for (unsigned char c : t.patterns[id]) {
                        node = t.transition(node, c);
                        if (node >= n) {
                            full = false;
                            break;
                        }
                    }
                    k += (full && node != 0 && t.terminal(node)) ? 1u : 0u;
                }
                spelled += k;
            });
        dictionary_language = dictionary_language && order.size() == n && terminal_paths == spelled;
    }
    im.dictionary_language = dictionary_language;
    im.path_id.assign(n, kKeep);
    if (dictionary_language) {
        for (uint32_t u = 0; u < n; ++u)
            if (unique_path[u]) im.path_id[u] = kNoId;
        std::vector<uint8_t> conflict(n, 0);
        // each pattern's (U, clean) in parallel, then applied in id order
        // (the outcome -- one id per U, or a conflict -- is order-independent)
        std::vector<uint32_t> claim_u(P, kNoId);
        std::vector<uint8_t> claim_clean(P, 0);
        parallel_slices(P, 4096, [&](size_t b, size_t e) {
            std::vector<uint32_t> path;
            for (size_t id = b; id < e; ++id) {
                path.assign(1, 0u);
                for (unsigned char c : t.patterns[id]) {
                    const uint32_t nx = t.transition(path.back(), c);
                    if (nx >= n) break;
                    path.push_back(nx);
                }
                const size_t L = path.size() - 1;
                if (L != t.patterns[id].size()) continue; // truncated away
                const uint32_t T = path[L];
                if (!t.terminal(T) || im.term_id[T] != kNoId) continue; // private terminals name themselves
                size_t u = L;
                while (u > 0 && !unique_path[path[u]]) --u;
                if (!unique_path[path[u]]) continue;
                bool clean = true;
                for (size_t i = u + 1; i < L; ++i) clean = clean && !t.terminal(path[i]);
                claim_u[id] = path[u];
                claim_clean[id] = clean ? 1u : 0u;
            }
        });
        for (size_t id = 0; id < P; ++id) {
            const uint32_t U = claim_u[id];
            if (U == kNoId) continue;
            if (!claim_clean[id] || (im.path_id[U] != kNoId && im.path_id[U] != uint32_t(id))) conflict[U] = 1;
            else im.path_id[U] = uint32_t(id);
        }
        for (uint32_t u = 0; u < n; ++u)
            if (conflict[u]) im.path_id[u] = kNoId;
    }
    // the path id a walk carries after entering node v from a parent carrying `pend`
    auto pend_at = [&](uint32_t v, uint32_t pend) { return im.path_id[v] != kKeep ? im.path_id[v] : pend; };

    // ---- buckets: CSR, each sorted by (length, id) -----------------------
    im.bucket_of.assign(n, kNoId);
    for (const auto& [node, ids] : t.buckets) {
        if (node >= n) continue;
        im.bucket_of[node] = uint32_t(im.bk_span.size() / 2);
        std::vector<uint32_t> sorted = ids;
        std::sort(sorted.begin(), sorted.end(), [&](uint32_t a, uint32_t b) {
            return im.pat_len[a] != im.pat_len[b] ? im.pat_len[a] < im.pat_len[b] : a < b;
        });
        im.bk_span.push_back(uint32_t(im.bk_entry.size() / 4));
        im.bk_span.push_back(uint32_t(sorted.size()));
        for (uint32_t id : sorted) {
            im.bk_entry.push_back(id);
            im.bk_entry.push_back(im.pat_len[id]);
            im.bk_entry.push_back(uint32_t(im.pat_off[id]));
            im.bk_entry.push_back(uint32_t(im.pat_off[id] >> 32));
        }
    }
    if (im.bk_span.empty()) im.bk_span.assign(2, 0);
    if (im.bk_entry.empty()) im.bk_entry.assign(4, 0);

    // ---- node records ------------------------------------------------------
    const uint32_t sigma = t.alphabet.size();
    im.groups = sigma <= 32 ? 0 : (sigma + 63) / 64;
    auto flags = [&](uint32_t u) {
        return (t.terminal(u) ? kFlagTerminal : 0u) | (im.bucket_of[u] != kNoId ? kFlagBucket : 0u);
    };
    if (im.groups == 0) {
        im.nodes.resize(size_t(n) * 2);
        parallel_slices(n, 1 << 16, [&](size_t b, size_t e) {
            for (size_t u = b; u < e; ++u) {
                im.nodes[2 * u] = t.cell(uint32_t(u))[0];
                im.nodes[2 * u + 1] = (kids[u] ? t.offset(uint32_t(u)) : 0u) | flags(uint32_t(u));
            }
        });
    } else {
        im.nodes.resize(size_t(n) * im.groups * 4);
        parallel_slices(n, 1 << 16, [&](size_t b, size_t e) {
            for (size_t u = b; u < e; ++u) {
                const uint32_t* c = t.cell(uint32_t(u));
                uint32_t base = kids[u] ? t.offset(uint32_t(u)) : 0u;
                for (uint32_t g = 0; g < im.groups; ++g) {
                    const uint32_t w0 = 2 * g < t.words ? c[2 * g] : 0u;
                    const uint32_t w1 = 2 * g + 1 < t.words ? c[2 * g + 1] : 0u;
                    uint32_t* r = &im.nodes[(u * im.groups + g) * 4];
                    r[0] = w0;
                    r[1] = w1;
                    r[2] = (base & kBaseMask) | flags(uint32_t(u));
                    r[3] = im.term_id[u];
                    base += uint32_t(__builtin_popcount(w0) + __builtin_popcount(w1));
                }
            }
        });
    }

    // ---- report depths: min_emit (BFS) -------------------------------------
    {
        std::vector<uint32_t> depth(n, UINT32_MAX), q{0};
        depth[0] = 0;
        uint32_t min_term = UINT32_MAX;
        for (size_t h = 0; h < q.size(); ++h) {
            const uint32_t u = q[h];
            if (u != 0 && t.terminal(u)) min_term = std::min(min_term, depth[u]);
            for (uint32_t i = 0; i < kids[u]; ++i) {
                const uint32_t c = t.offset(u) + i;
                if (depth[c] == UINT32_MAX) {
                    depth[c] = depth[u] + 1;
                    q.push_back(c);
                }
            }
        }
        im.min_emit = min_term;
        if (im.depth_limit && !t.buckets.empty()) im.min_emit = std::min(im.min_emit, im.depth_limit);
    }

    // ---- reach: longest root path (cyclic => unbounded), plus buckets ------
    if (im.depth_limit) {
        uint64_t r = im.depth_limit;
        for (const auto& [node, ids] : t.buckets)
            for (uint32_t id : ids) r = std::max<uint64_t>(r, im.pat_len[id]);
        im.reach = r;
    } else if (order.size() == n) {
        // acyclic (Kahn order covers every node): longest path in reverse
        // topological order
        std::vector<uint64_t> longest(n, 0);
        for (size_t h = n; h-- > 0;) {
            const uint32_t u = order[h];
            uint64_t best = 0;
            for (uint32_t k = 0; k < kids[u]; ++k) best = std::max(best, 1 + longest[t.offset(u) + k]);
            longest[u] = best;
        }
        im.reach = longest[0];
    } else {
        // iterative DFS post-order over the reachable graph
        std::vector<uint64_t> longest(n, 0);
        std::vector<uint8_t> state(n, 0); // 0 new, 1 on stack, 2 done
        std::vector<std::pair<uint32_t, uint32_t>> st{{0u, 0u}};
        state[0] = 1;
        bool cyclic = false;
        while (!st.empty() && !cyclic) {
            auto& [u, i] = st.back();
            if (i < kids[u]) {
                const uint32_t c = t.offset(u) + i++;
                if (state[c] == 1) cyclic = true;
                else if (state[c] == 0) {
                    state[c] = 1;
                    st.emplace_back(c, 0u);
                }
            } else {
                uint64_t best = 0;
                for (uint32_t k = 0; k < kids[u]; ++k) best = std::max(best, 1 + longest[t.offset(u) + k]);
                longest[u] = best;
                state[u] = 2;
                st.pop_back();
            }
        }
        im.reach = cyclic ? UINT64_MAX : longest[0];
    }

    // ---- start filter --------------------------------------------------------
    if (im.min_emit != UINT32_MAX) {
        const uint32_t k = std::min(im.min_emit, kMaxFilterKey);
        im.filter_k = k;
        std::vector<uint64_t> grams;
        std::vector<uint32_t> gram_node, gram_pend;
        const uint64_t cap = uint64_t(1) << 22;
        struct Frame {
            uint32_t node, depth;
            uint64_t key;
            uint32_t pend;
        };
        std::vector<Frame> st{{0u, 0u, 0ull, pend_at(0, kNoId)}};
        bool overflow = false;
        while (!st.empty() && !overflow) {
            Frame f = st.back();
            st.pop_back();
            if (f.depth == k) {
                grams.push_back(f.key);
                gram_node.push_back(f.node);
                gram_pend.push_back(f.pend);
                overflow = grams.size() > cap;
                continue;
            }
            const uint32_t* c = t.cell(f.node);
            uint32_t child = t.offset(f.node);
            for (uint32_t w = 0; w < t.words; ++w)
                for (uint32_t bits = c[w]; bits; bits &= bits - 1) {
                    const uint32_t s = w * 32 + uint32_t(__builtin_ctz(bits));
                    const uint64_t b = t.alphabet.byte_of(s);
                    st.push_back({child, f.depth + 1, f.key | (b << (8 * f.depth)), pend_at(child, f.pend)});
                    ++child;
                }
        }
        im.filter_paths = grams.size();
        if (grams.empty()) {
            im.min_emit = UINT32_MAX; // no start can reach a reporting depth
        } else if (!overflow) {
            auto popcount = [](const std::vector<uint32_t>& v) {
                uint64_t c = 0;
                for (uint32_t w : v) c += uint64_t(__builtin_popcount(w));
                return c;
            };
            // single-probe table over the whole k-byte key
            const uint32_t bits =
                std::clamp<uint32_t>(ceil_log2(grams.size()) + opt.filter_slack, 10, opt.max_filter_bits);
            std::vector<uint32_t> single((size_t(1) << bits) / 32, 0u);
            for (uint64_t g : grams) {
                const uint32_t k32 = filter_fold(g);
                single[filter_word(k32, bits - 5)] |= filter_mask_bit(k32);
            }
            double f_single = double(popcount(single)) / double(uint64_t(1) << bits);
            // pair table over the first 4 bytes (k >= 4)
            std::vector<uint32_t> pair;
            uint32_t pair_wb = 0;
            double f_pair = 1.0;
            if (k >= 4) {
                pair_wb = std::clamp<uint32_t>(ceil_log2(2 * grams.size()) + opt.filter_slack, 10, opt.max_filter_bits) - 5;
                pair.assign(size_t(1) << pair_wb, 0u);
                for (uint64_t g : grams) {
                    const uint32_t p = uint32_t(g); // p0 | p1 << 8 | p2 << 16 | p3 << 24
                    pair[pair_word(p >> 8, pair_wb)] |= filter_mask_bit(p & 0xFFu);        // role A
                    pair[pair_word(p & 0xFFFFFFu, pair_wb)] |= filter_mask_bit(p >> 24);   // role B
                }
                f_pair = double(popcount(pair)) / double(uint64_t(32) << pair_wb);
            }
            // Pass rates on text drawn uniformly from the alphabet (Monte Carlo,
            // fixed seed): what fraction of starts survive each level.
            double p_single = f_single, p_first = f_pair, p_both = f_pair * f_pair, p_true = 0.0;
            {
                const uint32_t sigma = t.alphabet.size();
                const uint32_t N = 1u << 15;
                uint64_t x = 0x9E3779B97F4A7C15ull;
                uint32_t n_single = 0, n_first = 0, n_both = 0, n_true = 0;
                std::vector<uint64_t> paths(grams);
                std::sort(paths.begin(), paths.end());
                auto word_bit = [](const std::vector<uint32_t>& tab, uint32_t word, uint32_t byte) {
                    return (tab[word] & filter_mask_bit(byte)) != 0;
                };
                for (uint32_t s = 0; s < N; ++s) {
                    uint64_t key = 0;
                    for (uint32_t b = 0; b < k; ++b) {
                        x ^= x << 13, x ^= x >> 7, x ^= x << 17;
                        key |= uint64_t(t.alphabet.byte_of(uint32_t(x % sigma))) << (8 * b);
                    }
                    const uint32_t k32 = filter_fold(key);
                    n_single += word_bit(single, filter_word(k32, bits - 5), k32);
                    n_true += std::binary_search(paths.begin(), paths.end(), key) ? 1u : 0u;
                    if (k >= 4) {
                        const uint32_t p = uint32_t(key);
                        const bool a = word_bit(pair, pair_word(p >> 8, pair_wb), p & 0xFFu);
                        const bool b = word_bit(pair, pair_word(p & 0xFFFFFFu, pair_wb), p >> 24);
                        n_first += (s & 1) ? a : b; // odd starts meet role A first
                        n_both += a && b;
                    }
                }
                p_single = double(n_single) / N;
                p_true = double(n_true) / N;
                if (k >= 4) p_first = double(n_first) / N, p_both = double(n_both) / N;
            }
            // Cost per start in issue slots (shared-memory wavefronts counted
            // like instructions): single = 6.75 SASS + 3.7 wavefronts; pair =
            // 4.75 + 1.85, plus a divergent second probe per first-level
            // survivor; each start reaching the walk queue costs ~60.
            const double cost_single = 10.45 + 60.0 * p_single;
            const double cost_pair = 6.6 + 30.0 * p_first + 60.0 * p_both;
            bool use_pair = k >= 4 && cost_pair < cost_single;
            f_single = p_single;
            f_pair = std::sqrt(p_both);
            if (opt.filter_mode == 1 || opt.filter_mode == 4) use_pair = false;
            if (opt.filter_mode == 2) use_pair = k >= 4;
            // Two-pass pipeline (lean filter pass, then the walking pass) for
            // the pair form: the walking pass re-checks survivors' first 4
            // bytes in shared memory.  (A single-probe filter pass was measured
            // slower than the fused kernel, c4 sigma=20: 1.22 against 1.26 TB/s,
            // and was removed.)
            if (use_pair) {
                const uint32_t kb = std::clamp<uint32_t>(ceil_log2(grams.size()) + opt.filter_slack, 10, 20);
                im.key4.assign((size_t(1) << kb) / 32, 0u);
                for (uint64_t g : grams) {
                    const uint32_t k32 = uint32_t(g);
                    im.key4[filter_word(k32, kb - 5)] |= filter_mask_bit(k32);
                }
            }
            if (use_pair) {
                im.filter_mode = 2;
                im.filter = std::move(pair);
                im.filter_bits = pair_wb + 5;
                im.pair_shift = 32 - pair_wb;
                im.filter_pass = p_both;
            } else {
                im.filter_mode = 1;
                im.filter = std::move(single);
                im.filter_bits = bits;
                im.filter_pass = p_single;
            }
            // Third level (L2-resident, whole k-byte key) when what reaches the
            // walk queue is still dense.
            // ... unless most of what passes are real depth-k paths (small
            // alphabets: DNA 14% of 16.6%): the jump table is exact, and one
            // more L2 round trip per survivor would filter almost nothing.
            const bool mostly_true = p_true > 0.5 * im.filter_pass;
            if ((im.filter_mode == 1 || im.filter_pass > 0.002) && !mostly_true) {
                const uint32_t bits2 =
                    std::clamp<uint32_t>(ceil_log2(grams.size()) + opt.filter2_slack, 16, opt.max_filter2_bits);
                im.filter2_bits = bits2;
                im.filter2.assign((size_t(1) << bits2) / 32, 0u);
                for (uint64_t g : grams) {
                    const uint32_t s2 = filter2_slot(filter_fold(g), bits2);
                    im.filter2[s2 >> 5] |= 1u << (s2 & 31);
                    // pair tries: a second bit in the same word (the hash's low
                    // bits) for the filter pass's two-bit test; single-bit
                    // probes of the same table stay conservative
                    if (im.filter_mode == 2) im.filter2[s2 >> 5] |= 1u << (filter2_hash(filter_fold(g)) & 31u);
                }
            }
            // Saturated first level (dictionaries of ~10^6 k-grams: 2^20 bits
            // in shared memory pass most random starts): the two-pass
            // pipeline with a filter pass that tests both levels for every
            // start (pfac_l2_filter_kernel), instead of the fused kernel's
            // one dependent L2 probe chain per survivor.
            if (im.filter_mode == 1 && k >= 4 && im.filter2_bits &&
                (opt.filter_mode == 4 || (opt.filter_mode == 0 && p_single > 0.25))) {
                im.filter_mode = 4;
                // its shared-memory level: 192 KiB (1.57 M bits, layout.hpp;
                // c5 1M: 47% of random starts pass instead of 61% with 2^20
                // bits), so fewer starts probe L2
                im.filter_l1.assign(kL1Words, 0u);
                for (uint64_t g : grams) {
                    const uint32_t k32 = filter_fold(g);
                    im.filter_l1[filter_l1_word(k32, kL1Words)] |= filter_mask_bit(k32);
                }
                const double f_l1 = double(popcount(im.filter_l1)) / double(uint64_t(32) * kL1Words);
                // a second bit per key in the same L2 word (from the hash's low
                // bits): the filter pass tests both with its one load (c5 1M:
                // 0.8% -> ~0.03% of its L2 probes pass); the fused kernel's
                // single-bit probe stays conservative
                for (uint64_t g : grams) {
                    const uint32_t h = filter2_hash(filter_fold(g));
                    im.filter2[(h >> (32 - im.filter2_bits)) >> 5] |= 1u << (h & 31u);
                }
                const double f2 = double(popcount(im.filter2)) / double(uint64_t(1) << im.filter2_bits);
                im.filter_pass = f_l1 * f2 * f2;
            }
            if (opt.jump) {
                std::vector<JumpEntry> entries(grams.size());
                for (size_t i = 0; i < grams.size(); ++i) {
                    const uint32_t node = gram_node[i];
                    const uint32_t b = im.bucket_of[node];
                    entries[i] = {uint32_t(grams[i]), uint32_t(grams[i] >> 32), node, im.term_id[node],
                                  b == kNoId ? 0u : im.bk_span[2 * size_t(b)],
                                  b == kNoId ? 0u : im.bk_span[2 * size_t(b) + 1],
                                  (t.terminal(node) ? 1u : 0u) | (b == kNoId ? 0u : 2u), gram_pend[i]};
                }
                std::vector<InlineList> lists;
                if (opt.jump_ext && im.dictionary_language) lists = inline_lists(t, im, entries, grams, k, 0);
                build_jump_table(im, entries, lists);
            }
        }
    }

    // ---- symbol-key mode (small alphabets) -----------------------------------
    // Byte keys carry log2(sigma) bits per byte: 8 bytes of DNA are 16 bits, of
    // a binary alphabet 8.  When the shortest report depth allows more than 8
    // symbols, keys are the first k symbols packed at 1/2/4 bits each, up to
    // 32 bits: sigma = 4 with 12-symbol keys has 24 bits of selectivity.  The
    // text is packed once per scan (pfac_pack_symbols_kernel) and scanned by
    // the symbol filter pass; the jump table is keyed the same way.
    {
        const uint32_t sigma = t.alphabet.size();
        // 4-bit symbols would need more than 8 of them (> 32-bit keys) to beat
        // byte keys, so symbol keys serve sigma <= 4
        const uint32_t sb = sigma <= 2 ? 1u : (sigma <= 4 ? 2u : 0u);
        const uint32_t ks = sb && im.min_emit != UINT32_MAX ? std::min(im.min_emit, 32u / sb) : 0u;
        if (opt.symbol_keys && sb && ks > std::min(im.min_emit, kMaxFilterKey) && opt.jump) {
            std::vector<uint32_t> keys, knode, kpend;
            struct SFrame {
                uint32_t node, depth, key, pend;
            };
            std::vector<SFrame> st{{0u, 0u, 0u, pend_at(0, kNoId)}};
            bool overflow = false;
            while (!st.empty() && !overflow) {
                const SFrame f = st.back();
                st.pop_back();
                if (f.depth == ks) {
                    keys.push_back(f.key);
                    knode.push_back(f.node);
                    kpend.push_back(f.pend);
                    overflow = keys.size() > (uint64_t(1) << 22);
                    continue;
                }
                const uint32_t* c = t.cell(f.node);
                uint32_t child = t.offset(f.node);
                for (uint32_t w = 0; w < t.words; ++w)
                    for (uint32_t bits = c[w]; bits; bits &= bits - 1) {
                        const uint32_t s = w * 32 + uint32_t(__builtin_ctz(bits));
                        st.push_back({child, f.depth + 1, f.key | (s << (sb * f.depth)), pend_at(child, f.pend)});
                        ++child;
                    }
            }
            if (!overflow && !keys.empty()) {
                im.filter_mode = 3;
                im.sym_bits = sb;
                im.filter_k = ks;
                im.filter_paths = keys.size();
                const uint32_t bits =
                    std::clamp<uint32_t>(ceil_log2(keys.size()) + opt.filter_slack, 10, opt.max_filter_bits);
                im.filter_bits = bits;
                im.filter.assign((size_t(1) << bits) / 32, 0u);
                for (uint32_t key : keys) im.filter[filter_word(key, bits - 5)] |= filter_mask_bit(key);
                // fraction of uniform random texts that survive: fill of the bitmap
                uint64_t set = 0;
                for (uint32_t w : im.filter) set += uint64_t(__builtin_popcount(w));
                im.filter_pass = double(set) / double(uint64_t(1) << bits);
                im.filter2_bits = 0;
                im.filter2.clear();
                // the walking pass re-checks candidates' packed keys under an
                // independent hash (filter2_hash first), like key4 for bytes,
                // when most filter survivors of random text would be false
                // positives (c4 sigma=4: +28%; sigma=2, where a random key is
                // a real path as often as a false positive, lost 3%)
                im.key4.clear();
                const double p_true = double(keys.size()) / std::ldexp(1.0, int(sb * ks));
                if (p_true < 0.25 * im.filter_pass) {
                    const uint32_t kb = std::clamp<uint32_t>(ceil_log2(keys.size()) + opt.filter_slack, 10, 20);
                    im.key4.assign((size_t(1) << kb) / 32, 0u);
                    for (uint32_t key : keys) {
                        const uint32_t h = filter2_hash(key);
                        im.key4[filter_word(h, kb - 5)] |= filter_mask_bit(h);
                    }
                }
                std::vector<JumpEntry> entries(keys.size());
                for (size_t i = 0; i < keys.size(); ++i) {
                    const uint32_t node = knode[i];
                    const uint32_t b = im.bucket_of[node];
                    entries[i] = {keys[i], 0u, node, im.term_id[node],
                                  b == kNoId ? 0u : im.bk_span[2 * size_t(b)],
                                  b == kNoId ? 0u : im.bk_span[2 * size_t(b) + 1],
                                  (t.terminal(node) ? 1u : 0u) | (b == kNoId ? 0u : 2u), kpend[i]};
                }
                std::vector<InlineList> lists;
                if (opt.jump_ext && im.dictionary_language)
                    lists = inline_lists(t, im, entries, std::vector<uint64_t>(keys.begin(), keys.end()), ks, sb);
                build_jump_table(im, entries, lists);
            }
        }
    }
    // ---- direct-index form (filter mode 5, layout.hpp) -------------------------
    // Alphabets of at most 4 symbols whose every pattern has 8..32 symbols
    // (c2: DNA, 10k patterns of 8-32): the byte-key path filters on 8-byte
    // keys hashed into a bitmap and then, per surviving start, reads a jump
    // slot and its inline list from L2 (two dependent round trips for the 14%
    // of random DNA starts that are real 8-symbol prefixes).  Here the 16-bit
    // key of 8 packed symbols indexes exact tables in shared memory and the
    // start's patterns are compared 2 bits per symbol, with no L2 round trip.
    if (opt.dna && im.filter_mode != 3 && im.dictionary_language && t.alphabet.size() <= 4 && P > 0 && P <= 65535) {
        struct E {
            uint32_t key, len, id;
            uint64_t sym;
        };
        std::vector<E> es;
        es.reserve(P);
        bool ok = true;
        for (size_t id = 0; id < P && ok; ++id) {
            const auto& pat = t.patterns[id];
            if (pat.size() < kDnaK || pat.size() > kDnaMaxLen) {
                ok = false;
                break;
            }
            uint64_t sym = 0;
            for (size_t i = 0; i < pat.size(); ++i) {
                const int s = t.alphabet.symbol_of(uint8_t(pat[i]));
                if (s < 0) ok = false;
                sym |= uint64_t(uint32_t(s) & 3u) << (2 * i);
            }
            es.push_back({uint32_t(sym & 0xFFFFu), uint32_t(pat.size()), uint32_t(id), sym});
        }
        if (ok) {
            std::sort(es.begin(), es.end(), [](const E& x, const E& y) {
                return x.key != y.key ? x.key < y.key : (x.len != y.len ? x.len < y.len : x.id < y.id);
            });
            std::vector<uint32_t> first;
            std::vector<uint32_t> bitmap(2048, 0u);
            for (size_t i = 0; i < es.size(); ++i) {
                if (i == 0 || es[i].key != es[i - 1].key) {
                    if (!first.empty() && i - first.back() > kDnaMaxPerKey) ok = false;
                    first.push_back(uint32_t(i));
                    bitmap[es[i].key >> 5] |= 1u << (es[i].key & 31u);
                }
            }
            if (!first.empty() && es.size() - first.back() > kDnaMaxPerKey) ok = false;
            const uint32_t nk = uint32_t(first.size());
            first.push_back(uint32_t(es.size()));
            const uint32_t bytes = dna_blob_bytes(nk, uint32_t(P));
            if (ok && bytes <= kDnaMaxBlob) {
                std::vector<uint8_t> blob(bytes, 0);
                std::memcpy(blob.data(), bitmap.data(), 2048 * 4);
                uint32_t run = 0;
                for (uint32_t w = 0; w < 2048; ++w) {
                    const uint16_t r = uint16_t(run);
                    std::memcpy(blob.data() + kDnaWrankOff + 2 * w, &r, 2);
                    run += uint32_t(__builtin_popcount(bitmap[w]));
                }
                for (uint32_t r = 0; r <= nk; ++r) {
                    const uint16_t f = uint16_t(first[r]);
                    std::memcpy(blob.data() + kDnaFirstOff + 2 * r, &f, 2);
                }
                for (size_t i = 0; i < es.size(); ++i) {
                    std::memcpy(blob.data() + dna_sym_off(nk) + 8 * i, &es[i].sym, 8);
                    const uint32_t meta = (es[i].len << 16) | es[i].id;
                    std::memcpy(blob.data() + dna_meta_off(nk, uint32_t(P)) + 4 * i, &meta, 4);
                }
                im.dna.assign(bytes / 4, 0u);
                std::memcpy(im.dna.data(), blob.data(), bytes);
                im.dna_keys = nk;
                im.dna_pats = uint32_t(P);
                im.filter_mode = 5;
                im.filter_pass = double(nk) / 65536.0;
            }
        }
    }

    if (im.filter.empty()) im.filter.push_back(0);
    if (im.filter2.empty()) im.filter2.push_back(0);
    if (im.jump.empty()) im.jump.assign(kJumpWords, 0u), im.jump_ext.clear();

    for (uint32_t u = 0; u < n; ++u)
        if (t.terminal(u) && u != 0) (im.term_id[u] == kNoId ? im.keyed_terminals : im.private_terminals)++;
    return im;
}

} // namespace hfb

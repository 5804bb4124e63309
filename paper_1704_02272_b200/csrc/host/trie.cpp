// trie.cpp -- the host trie compiler: canonical bitmap trie, compression
// stages and prefix truncation.
//
// The canonical layout is an API-visible artefact (node indices come back
// from hepfac_trie_transition, node counts and .htri bytes are compared by
// callers), so its placement rules follow the reference exactly:
//   - node = ceil(sigma/32) bitmap words + offset word (MSB terminal)
//     (reference trie.hpp:45-59);
//   - breadth-first, first-reference placement; a multi-child run is
//     consecutive and an already-placed node inside a run gets a shallow copy
//     slot (trie.cpp:133-217);
//   - stage 1 / stage 2 / truncation rewrite rules (compression.cpp:58-176,
//     prefix.cpp:14-51).
// The construction itself is different: stage-0 tries are built level by
// level from the symbol-sorted pattern list (no pointer graph, no queue),
// and rewrites operate on a flat CSR graph.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <numeric>
#include <thread>
#include <unordered_map>

#include "core.hpp"

namespace hfb {

unsigned compiler_threads()
{
    if (const char* s = std::getenv("HEPFAC_COMPILER_THREADS")) {
        const long v = std::strtol(s, nullptr, 10);
        if (v >= 1 && v <= 1024) return unsigned(v);
    }
    return std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
}

namespace {

// Stable order of `v` under `less`, sorted in parallel slices and merged
// pairwise (the result equals std::stable_sort's).
template <typename T, typename Less>
void parallel_sort(std::vector<T>& v, Less less)
{
    const size_t n = v.size();
    const unsigned t = unsigned(std::min<size_t>(compiler_threads(), std::max<size_t>(1, n / 65536)));
    if (t <= 1) {
        std::stable_sort(v.begin(), v.end(), less);
        return;
    }
    std::vector<size_t> cut(t + 1);
    for (unsigned i = 0; i <= t; ++i) cut[i] = n * i / t;
    parallel_slices(t, 1, [&](size_t b, size_t e) {
        for (size_t i = b; i < e; ++i) std::stable_sort(v.begin() + cut[i], v.begin() + cut[i + 1], less);
    });
    for (size_t width = 1; width < t; width *= 2) {
        std::vector<std::thread> pool;
        for (size_t i = 0; i + width < t; i += 2 * width) {
            const size_t lo = cut[i], mid = cut[i + width], hi = cut[std::min<size_t>(t, i + 2 * width)];
            pool.emplace_back([&, lo, mid, hi] { std::inplace_merge(v.begin() + lo, v.begin() + mid, v.begin() + hi, less); });
        }
        for (auto& th : pool) th.join();
    }
}

} // namespace

std::string format_mib(uint64_t bytes)
{
    uint64_t tenths = (bytes * 10) >> 20; // truncated, not rounded
    return std::to_string(tenths / 10) + "." + std::to_string(tenths % 10);
}

double reduction_percent(uint64_t before, uint64_t after)
{
    return after == 0 ? 0.0 : 100.0 * double(before - after) / double(after);
}

uint32_t Trie::child_count(uint32_t n) const
{
    const uint32_t* c = cell(n);
    uint32_t k = 0;
    for (uint32_t i = 0; i < words; ++i) k += uint32_t(__builtin_popcount(c[i]));
    return k;
}

uint32_t Trie::transition(uint32_t node, uint8_t byte) const
{
    int s = alphabet.symbol_of(byte);
    if (s < 0) return kNone;
    const uint32_t* c = cell(node);
    const uint32_t w = uint32_t(s) >> 5, bit = 1u << (uint32_t(s) & 31u);
    if (!(c[w] & bit)) return kNone;
    uint32_t rank = uint32_t(__builtin_popcount(c[w] & (bit - 1)));
    for (uint32_t i = 0; i < w; ++i) rank += uint32_t(__builtin_popcount(c[i]));
    return (c[words] & kOffsetMask) + rank;
}

void Trie::set_lengths()
{
    min_len = max_len = 0;
    for (const auto& p : patterns) {
        uint32_t l = uint32_t(p.size());
        if (min_len == 0 || l < min_len) min_len = l;
        max_len = std::max(max_len, l);
    }
}

// ---------------------------------------------------------------------------
// Stage-0 construction.
//
// In a tree laid out breadth-first with children in symbol order, the nodes of
// depth d appear in lexicographic (symbol-wise) order of the prefixes they
// spell.  So sorting the patterns once and sweeping depth by depth numbers
// every node directly: a new node starts wherever (parent, symbol) changes
// along the sorted list.
std::unique_ptr<Trie> build_trie(const PatternSet& set)
{
    if (set.patterns.empty()) invalid("empty pattern set");
    for (const auto& p : set.patterns)
        if (p.size() > 65535) invalid("pattern longer than 65535 bytes");

    const Alphabet& a = set.alphabet;
    const size_t n = set.patterns.size();
    std::vector<std::string> keys(n); // symbol-index strings: byte order == symbol order
    parallel_slices(n, 16384, [&](size_t b, size_t e) {
        for (size_t i = b; i < e; ++i) {
            const std::string& p = set.patterns[i];
            keys[i].resize(p.size());
            for (size_t j = 0; j < p.size(); ++j) keys[i][j] = char(a.symbol_of(uint8_t(p[j])));
        }
    });
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    // patterns are distinct, so any sort gives the same order
    parallel_sort(order, [&](uint32_t x, uint32_t y) { return keys[x] < keys[y]; });

    auto t = std::make_unique<Trie>(a);
    const uint32_t stride = t->stride();
    CellVector& cells = t->cells;
    cells.assign(stride, 0); // root
    uint64_t nodes = 1;

    std::vector<uint32_t> active(order); // patterns still longer than the current depth
    std::vector<uint32_t> at(n, 0);      // node currently reached by each pattern
    std::vector<uint32_t> next_active;
    for (uint32_t depth = 0; !active.empty(); ++depth) {
        next_active.clear();
        uint32_t last_parent = Trie::kNone, last_sym = Trie::kNone, last_node = 0;
        for (uint32_t i : active) {
            const uint32_t parent = at[i];
            const uint32_t sym = uint8_t(keys[i][depth]);
            if (parent != last_parent || sym != last_sym) {
                if (nodes >= Trie::kMaxNodes) invalid("trie too large");
                last_node = uint32_t(nodes++);
                cells.resize(size_t(nodes) * stride, 0);
                uint32_t* pc = cells.data() + size_t(parent) * stride;
                bool first_child = true;
                for (uint32_t w = 0; w < t->words; ++w) first_child = first_child && pc[w] == 0;
                if (first_child) pc[t->words] = (pc[t->words] & Trie::kTerminal) | last_node;
                pc[sym >> 5] |= 1u << (sym & 31u);
                last_parent = parent;
                last_sym = sym;
            }
            at[i] = last_node;
            if (keys[i].size() == depth + 1)
                cells[size_t(last_node) * stride + t->words] |= Trie::kTerminal;
            else
                next_active.push_back(i);
        }
        active.swap(next_active);
    }
    t->node_count = uint32_t(nodes);
    t->patterns = set.patterns;
    t->set_lengths();
    return t;
}

// ---------------------------------------------------------------------------
// Flat graph form used by the rewrite passes.  Node ids are the source trie's
// array indices; each node owns a contiguous edge range (symbol ascending).

namespace {

struct Graph {
    std::vector<uint32_t> first, degree; // edge range per node
    std::vector<uint16_t> sym;
    std::vector<uint32_t> dst;
    std::vector<uint8_t> term;

    uint32_t size() const { return uint32_t(first.size()); }
    uint32_t only_child(uint32_t u) const { return dst[first[u]]; }
};

Graph graph_of(const Trie& t)
{
    Graph g;
    const uint32_t n = t.node_count;
    g.first.resize(n);
    g.degree.resize(n);
    g.term.resize(n);
    // degrees, then edge offsets by a prefix sum, then the edges: each pass
    // on all host threads
    parallel_slices(n, 1 << 16, [&](size_t b, size_t e) {
        for (size_t u = b; u < e; ++u) {
            g.degree[u] = t.child_count(uint32_t(u));
            g.term[u] = (t.cell(uint32_t(u))[t.words] & Trie::kTerminal) ? 1 : 0;
        }
    });
    size_t edges = 0;
    for (uint32_t u = 0; u < n; ++u) {
        g.first[u] = uint32_t(edges);
        edges += g.degree[u];
    }
    g.sym.resize(edges);
    g.dst.resize(edges);
    parallel_slices(n, 1 << 16, [&](size_t b, size_t e) {
        for (size_t u = b; u < e; ++u) {
            const uint32_t* c = t.cell(uint32_t(u));
            uint32_t target = c[t.words] & Trie::kOffsetMask;
            size_t at = g.first[u];
            for (uint32_t w = 0; w < t.words; ++w) {
                uint32_t bits = c[w];
                while (bits) {
                    const uint32_t bit = uint32_t(__builtin_ctz(bits));
                    bits &= bits - 1;
                    g.sym[at] = uint16_t(w * 32 + bit);
                    g.dst[at++] = target++;
                }
            }
        }
    });
    return g;
}

// Breadth-first first-reference emission (the reference's TrieAssembler rule,
// trie.cpp:133-217): slots are appended in BFS order; a multi-child node's
// children take one consecutive run, where an already-placed child becomes a
// copy slot; a single child is linked to its primary slot; every node's
// primary slot is its first reference in BFS order.
//
// Here the queue is processed a whole BFS level at a time, on all host
// threads.  The slots of level l+1 are created by the references of level
// l's slots, in (slot, edge) order, so "first reference" is the minimum
// reference index among a child's references in the level (an atomic
// minimum), and a prefix sum over the heads numbers the new slots.  The
// result is identical to the one-slot-at-a-time queue.
// `bucket_src` (optional) maps source node -> pattern ids; keys are remapped to
// the emitted primary slots.
std::unique_ptr<Trie> emit(const Graph& g, const Trie& like, Stage stage,
                           std::optional<uint32_t> depth_limit,
                           const std::vector<std::pair<uint32_t, std::vector<uint32_t>>>* bucket_src)
{
    constexpr uint32_t kUnplaced = Trie::kNone;
    constexpr size_t kGrain = 1 << 14;
    std::vector<uint32_t> slot_of_node(g.size(), kUnplaced); // primary slot per graph node
    // minimum reference index of each node in the level that places it (a
    // node is referenced while unplaced in exactly one level: its first
    // reference places it)
    std::vector<uint32_t> first_ref(g.size(), kUnplaced);
    std::vector<uint32_t> node_of_slot{0};
    std::vector<uint8_t> copy_slot{0};
    std::vector<uint32_t> child_base{0};
    slot_of_node[0] = 0;
    // every slot but the root is made by one reference (edge) of a slot
    const size_t max_slots = std::min<size_t>(size_t(Trie::kMaxNodes), g.dst.size() + 1);
    node_of_slot.reserve(max_slots);
    copy_slot.reserve(max_slots);
    child_base.reserve(max_slots);

    std::vector<uint64_t> ref_base, made; // per head of the level: first reference, first new slot
    std::vector<uint8_t> prim;            // per reference of the level: places its child's primary
    for (size_t h0 = 0; h0 < node_of_slot.size();) {
        const size_t h1 = node_of_slot.size(), L = h1 - h0;
        auto degree = [&](size_t i) -> uint32_t { return copy_slot[h0 + i] ? 0u : g.degree[node_of_slot[h0 + i]]; };
        ref_base.assign(L + 1, 0);
        for (size_t i = 0; i < L; ++i) ref_base[i + 1] = ref_base[i] + degree(i);
        const uint64_t R = ref_base[L];
        if (R >= kUnplaced) fail(HEPFAC_ERR_INTERNAL, "trie level exceeds 2^32 references");
        // 1. first reference of every unplaced child
        parallel_slices(L, kGrain, [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) {
                const uint32_t d = degree(i);
                const uint32_t f = d ? g.first[node_of_slot[h0 + i]] : 0u;
                for (uint32_t k = 0; k < d; ++k) {
                    const uint32_t c = g.dst[f + k];
                    if (slot_of_node[c] != kUnplaced) continue;
                    const uint32_t r = uint32_t(ref_base[i] + k);
                    std::atomic_ref<uint32_t> m(first_ref[c]);
                    uint32_t cur = m.load(std::memory_order_relaxed);
                    while (r < cur && !m.compare_exchange_weak(cur, r, std::memory_order_relaxed)) {
                    }
                }
            }
        });
        // 2. which references place a primary, and how many slots each head makes
        prim.assign(size_t(R), 0);
        made.assign(L + 1, 0);
        parallel_slices(L, kGrain, [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) {
                const uint32_t d = degree(i);
                const uint32_t f = d ? g.first[node_of_slot[h0 + i]] : 0u;
                for (uint32_t k = 0; k < d; ++k) {
                    const uint32_t c = g.dst[f + k];
                    prim[ref_base[i] + k] = slot_of_node[c] == kUnplaced && first_ref[c] == uint32_t(ref_base[i] + k);
                }
                made[i + 1] = d > 1 ? d : (d == 1 ? prim[ref_base[i]] : 0u);
            }
        });
        for (size_t i = 0; i < L; ++i) made[i + 1] += made[i];
        const uint64_t total = h1 + made[L];
        if (total > Trie::kMaxNodes) fail(HEPFAC_ERR_INTERNAL, "trie exceeds 2^31-1 nodes");
        node_of_slot.resize(total);
        copy_slot.resize(total);
        child_base.resize(total, 0);
        // 3. create the level's slots; single children placed here are linked
        parallel_slices(L, kGrain, [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) {
                const uint32_t d = degree(i);
                if (d == 0) continue;
                const uint32_t f = g.first[node_of_slot[h0 + i]];
                const uint32_t base = uint32_t(h1 + made[i]);
                if (d == 1 && !prim[ref_base[i]]) continue; // linked in step 4
                child_base[h0 + i] = base;
                for (uint32_t k = 0; k < d; ++k) {
                    const uint32_t c = g.dst[f + k], slot = base + k;
                    const bool p = prim[ref_base[i] + k];
                    node_of_slot[slot] = c;
                    copy_slot[slot] = p ? 0 : 1;
                    if (p) slot_of_node[c] = slot;
                }
            }
        });
        // 4. single children placed earlier, or by another head of this level
        parallel_slices(L, kGrain, [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i)
                if (degree(i) == 1 && !prim[ref_base[i]])
                    child_base[h0 + i] = slot_of_node[g.dst[g.first[node_of_slot[h0 + i]]]];
        });
        h0 = h1;
    }

    auto t = std::make_unique<Trie>(like.alphabet);
    t->node_count = uint32_t(node_of_slot.size());
    const uint32_t stride = t->stride();
    t->cells.resize(size_t(t->node_count) * stride); // uninitialised: every word is written below
    parallel_slices(t->node_count, 1 << 16, [&](size_t b, size_t e) {
        for (size_t s = b; s < e; ++s) {
            const uint32_t u = node_of_slot[s];
            uint32_t* c = t->cells.data() + s * stride;
            std::fill(c, c + t->words, 0u);
            for (uint32_t e2 = g.first[u]; e2 < g.first[u] + g.degree[u]; ++e2)
                c[g.sym[e2] >> 5] |= 1u << (g.sym[e2] & 31u);
            const uint32_t src = copy_slot[s] ? slot_of_node[u] : uint32_t(s);
            c[t->words] = (child_base[src] & Trie::kOffsetMask) | (g.term[u] ? Trie::kTerminal : 0u);
        }
    });
    t->patterns = like.patterns;
    t->set_lengths();
    t->stage = stage;
    t->depth_limit = depth_limit;
    if (bucket_src) {
        for (const auto& [u, ids] : *bucket_src) {
            if (slot_of_node[u] == kUnplaced) continue;
            auto sorted = ids;
            std::sort(sorted.begin(), sorted.end());
            t->buckets.emplace_back(slot_of_node[u], std::move(sorted));
        }
        std::sort(t->buckets.begin(), t->buckets.end(),
                  [](const auto& x, const auto& y) { return x.first < y.first; });
    }
    return t;
}

} // namespace

// ---------------------------------------------------------------------------
// Stage 1 (reference compression.cpp:58-94): every childless terminal below a
// unary parent is redirected to one shared terminal, the lowest-indexed
// childless terminal.  Multi-child parents keep private leaves because two
// slots of one run cannot alias a single cell (compression.hpp:26-31).
std::unique_ptr<Trie> merge_final_nodes(const Trie& t, CompressionStats* stats)
{
    if (t.stage != Stage::None) fail(HEPFAC_ERR_STATE, "trie is already compressed");
    if (t.depth_limit) invalid("cannot compress a truncated trie");
    Graph g = graph_of(t);
    uint32_t shared = Trie::kNone;
    for (uint32_t u = 0; u < g.size() && shared == Trie::kNone; ++u)
        if (g.term[u] && g.degree[u] == 0) shared = u;
    if (shared != Trie::kNone)
        for (uint32_t u = 0; u < g.size(); ++u) {
            if (g.degree[u] != 1) continue;
            uint32_t& c = g.dst[g.first[u]];
            if (g.term[c] && g.degree[c] == 0) c = shared;
        }
    auto out = emit(g, t, Stage::FinalMerged, std::nullopt, nullptr);
    if (stats) {
        stats->nodes_before = t.node_count;
        stats->nodes_after_stage1 = stats->nodes_after_stage2 = out->node_count;
        stats->pattern_count = t.patterns.size();
        stats->reduction_percent = reduction_percent(t.node_count, out->node_count);
    }
    return out;
}

// ---------------------------------------------------------------------------
// Stage 2 (reference compression.cpp:96-176): tails of up to three unary,
// non-terminal nodes ending in a shared terminal are merged into one class
// representative per suffix string.
std::unique_ptr<Trie> merge_tail_chains(const Trie& t, CompressionStats* stats)
{
    if (t.stage != Stage::FinalMerged) fail(HEPFAC_ERR_STATE, "tail merge requires stage-1 output");
    Graph g = graph_of(t);
    const Alphabet& a = t.alphabet;

    auto child_by_sym = [&](uint32_t u, uint32_t s) { // edges are symbol-ascending
        const auto b = g.sym.begin() + g.first[u], e = b + g.degree[u];
        const auto it = std::lower_bound(b, e, uint16_t(s));
        return (it != e && *it == s) ? g.dst[size_t(it - g.sym.begin())] : Trie::kNone;
    };
    auto leaf_terminal = [&](uint32_t u) { return g.term[u] && g.degree[u] == 0; };
    // A suffix of k <= 3 raw bytes, tagged with k, packed into 32 bits.
    auto suffix_key = [](const std::string& p, uint32_t k) {
        uint32_t key = k << 24;
        for (uint32_t i = 0; i < k; ++i) key |= uint32_t(uint8_t(p[p.size() - k + i])) << (8 * (2 - i));
        return key;
    };

    // suffix -> representative node, directly indexed (2^24 + 2^16 + 2^8 slots)
    auto suffix_index = [](uint32_t key) -> size_t {
        const uint32_t k = key >> 24;
        if (k == 3) return key & 0xFFFFFFu;
        if (k == 2) return (size_t(1) << 24) + ((key >> 8) & 0xFFFFu);
        return (size_t(1) << 24) + (size_t(1) << 16) + ((key >> 16) & 0xFFu);
    };
    std::vector<uint32_t> rep_of_suffix((size_t(1) << 24) + (size_t(1) << 16) + 256, Trie::kNone);
    std::vector<std::pair<uint32_t, uint32_t>> reps;      // (node, suffix) in creation order
    std::vector<std::pair<uint32_t, uint32_t>> rewires;   // (parent, new only child)
    // Phase A (parallel, per pattern): its path's last nodes and the length
    // of its eligible tail chain.  Phase B (serial, pattern order) assigns the
    // class representatives, which depends on which pattern comes first.
    struct Tail {
        uint32_t chain = 0;
        uint32_t node[5] = {0, 0, 0, 0, 0}; // path[L - k] for k = 0..4
    };
    const size_t P = t.patterns.size();
    std::vector<Tail> tails(P);
    std::vector<uint8_t> missing(P, 0);
    parallel_slices(P, 8192, [&](size_t b, size_t e) {
        std::vector<uint32_t> path;
        for (size_t i = b; i < e; ++i) {
            const std::string& p = t.patterns[i];
            const uint32_t L = uint32_t(p.size());
            if (L < 4) continue;
            path.assign(1, 0u);
            for (unsigned char ch : p) {
                const uint32_t nx = child_by_sym(path.back(), uint32_t(a.symbol_of(ch)));
                if (nx == Trie::kNone) {
                    missing[i] = 1;
                    break;
                }
                path.push_back(nx);
            }
            if (missing[i]) continue;
            // Longest eligible chain: path[L-k] unary & non-terminal, the
            // deepest one pointing at a shared (leaf) terminal.
            uint32_t chain = 0;
            for (uint32_t k = 1; k <= 3; ++k) {
                const uint32_t v = path[L - k];
                if (g.term[v] || g.degree[v] != 1) break;
                if (k == 1 && !leaf_terminal(g.only_child(v))) break;
                chain = k;
            }
            // The edge into the chain head must belong to a unary parent.
            while (chain >= 1 && g.degree[path[L - chain - 1]] > 1) --chain;
            tails[i].chain = chain;
            for (uint32_t k = 0; k <= 4; ++k) tails[i].node[k] = path[L - k];
        }
    });
    for (size_t i = 0; i < P; ++i)
        if (missing[i]) fail(HEPFAC_ERR_INTERNAL, "pattern missing from trie");

    for (size_t i = 0; i < P; ++i) {
        const std::string& p = t.patterns[i];
        const uint32_t chain = tails[i].chain;
        if (chain == 0) continue;
        const uint32_t* node = tails[i].node; // node[k] = path[L - k]
        uint32_t replace = 0; // deepest level whose class already has another owner
        for (uint32_t k = chain; k >= 1; --k) {
            const uint32_t rep = rep_of_suffix[suffix_index(suffix_key(p, k))];
            if (rep != Trie::kNone && rep != node[k]) {
                replace = k;
                break;
            }
        }
        for (uint32_t k = replace + 1; k <= chain; ++k) {
            const uint32_t key = suffix_key(p, k);
            uint32_t& rep = rep_of_suffix[suffix_index(key)];
            if (rep == Trie::kNone) rep = node[k], reps.emplace_back(node[k], key);
        }
        if (replace >= 1)
            rewires.emplace_back(node[replace + 1], rep_of_suffix[suffix_index(suffix_key(p, replace))]);
    }

    // Representatives of k-suffixes point at the representative of their
    // (k-1)-suffix, then replaced chains are cut over.
    for (const auto& [node, key] : reps) {
        const uint32_t k = key >> 24;
        if (k < 2) continue;
        // drop the first byte: shift the remaining k-1 bytes up one position
        const uint32_t sub = ((k - 1) << 24) | ((key << 8) & 0x00FFFF00u);
        const uint32_t rep = rep_of_suffix[suffix_index(sub)];
        if (rep != Trie::kNone) g.dst[g.first[node]] = rep;
    }
    for (const auto& [parent, child] : rewires) g.dst[g.first[parent]] = child;

    auto out = emit(g, t, Stage::TailMerged, std::nullopt, nullptr);
    if (stats) {
        stats->nodes_before = t.node_count;
        stats->nodes_after_stage1 = t.node_count;
        stats->nodes_after_stage2 = out->node_count;
        stats->pattern_count = t.patterns.size();
        stats->reduction_percent = reduction_percent(t.node_count, out->node_count);
    }
    return out;
}

// ---------------------------------------------------------------------------
// Truncation (reference prefix.cpp:14-51).

std::vector<uint32_t> first_reach_depths(const Trie& t)
{
    std::vector<uint32_t> depth(t.node_count, Trie::kNone);
    std::vector<uint32_t> frontier{0}, next;
    depth[0] = 0;
    for (uint32_t d = 0; !frontier.empty(); ++d) {
        next.clear();
        for (uint32_t u : frontier) {
            const uint32_t k = t.child_count(u), base = t.offset(u);
            for (uint32_t i = 0; i < k; ++i)
                if (depth[base + i] == Trie::kNone) {
                    depth[base + i] = d + 1;
                    next.push_back(base + i);
                }
        }
        frontier.swap(next);
    }
    return depth;
}

std::vector<std::pair<uint32_t, std::vector<uint32_t>>> verification_buckets(const Trie& t,
                                                                              uint32_t depth)
{
    std::unordered_map<uint32_t, std::vector<uint32_t>> by_node;
    for (uint32_t id = 0; id < t.patterns.size(); ++id) {
        const std::string& p = t.patterns[id];
        if (p.size() <= depth) continue;
        uint32_t node = 0;
        for (uint32_t i = 0; i < depth; ++i) {
            node = t.transition(node, uint8_t(p[i]));
            if (node >= t.node_count) fail(HEPFAC_ERR_INTERNAL, "dictionary pattern not present in trie");
        }
        by_node[node].push_back(id); // ids arrive ascending
    }
    std::vector<std::pair<uint32_t, std::vector<uint32_t>>> out(by_node.begin(), by_node.end());
    std::sort(out.begin(), out.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    return out;
}

static std::unique_ptr<Trie> clone(const Trie& t)
{
    auto c = std::make_unique<Trie>(t.alphabet);
    c->node_count = t.node_count;
    c->cells = t.cells;
    c->patterns = t.patterns;
    c->min_len = t.min_len;
    c->max_len = t.max_len;
    c->stage = t.stage;
    c->depth_limit = t.depth_limit;
    c->buckets = t.buckets;
    c->loaded = t.loaded;
    return c;
}

std::unique_ptr<Trie> truncate_trie(const Trie& t, uint32_t depth, bool* was_noop)
{
    if (depth == 0) invalid("truncation depth must be >= 1");
    if (t.stage == Stage::TailMerged) fail(HEPFAC_ERR_STATE, "cannot truncate a tail-merged trie");
    if (t.depth_limit) fail(HEPFAC_ERR_STATE, "trie is already truncated");
    if (depth >= t.max_len) {
        if (was_noop) *was_noop = true;
        return clone(t);
    }
    Graph g = graph_of(t);
    const auto depths = first_reach_depths(t);
    for (uint32_t u = 0; u < g.size(); ++u)
        if (depths[u] >= depth) g.degree[u] = 0;
    const auto buckets = verification_buckets(t, depth);
    auto out = emit(g, t, t.stage, depth, &buckets);
    if (was_noop) *was_noop = false;
    return out;
}

} // namespace hfb

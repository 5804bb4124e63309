// core.hpp -- host-side data model of the B200 PFAC library.
//
// Everything in this header is the "trie compiler" side of the drop-in
// boundary: alphabets, pattern sets, the canonical bitmap
// trie (the reference's exact cell layout, because node indices, node counts
// and .htri bytes are observable through the C ABI), compression stages,
// truncation and the .htri codec.  The match path itself runs on the GPU
// (csrc/cuda/); nothing here scans text.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "hepfac.h"

namespace hfb {

// Typed failure carrying the C status it maps to.  Messages reproduce the
// reference's wording (its capi.cpp:39-64 classifies by message substring,
// callers may print hepfac_last_error()).
struct Error : std::runtime_error {
    hepfac_status_t status;
    Error(hepfac_status_t s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(hepfac_status_t s, const std::string& msg) { throw Error(s, msg); }
[[noreturn]] inline void invalid(const std::string& msg) { fail(HEPFAC_ERR_INVALID_ARG, msg); }

std::string hex_byte(uint8_t b); // "0x4a"-style suffix helper: returns "4a"

// Host compiler threads: HEPFAC_COMPILER_THREADS, else the hardware threads
// (at most 64).
unsigned compiler_threads();

// fn(begin, end) over [0, n) in contiguous slices, one per thread; serial
// below `grain` items.  Results must not depend on the slicing.
template <typename Fn>
void parallel_slices(size_t n, size_t grain, Fn&& fn)
{
    const unsigned t = unsigned(std::min<size_t>(compiler_threads(), std::max<size_t>(1, n / std::max<size_t>(grain, 1))));
    if (t <= 1) {
        fn(size_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(t);
    for (unsigned i = 0; i < t; ++i)
        pool.emplace_back([&, i] { fn(n * i / t, n * (i + 1) / t); });
    for (auto& th : pool) th.join();
}

// Vector whose resize(n) leaves the new elements uninitialised, so a large
// trie's cells are first touched (and paged in) by the threads that fill them.
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = DefaultInitAlloc<U>;
    };
    DefaultInitAlloc() = default;
    template <class U>
    DefaultInitAlloc(const DefaultInitAlloc<U>&) noexcept {}
    template <class U>
    void construct(U* p) noexcept { ::new (static_cast<void*>(p)) U; }
    template <class U, class... A>
    void construct(U* p, A&&... a) { ::new (static_cast<void*>(p)) U(std::forward<A>(a)...); }
};
using CellVector = std::vector<uint32_t, DefaultInitAlloc<uint32_t>>;

// ---------------------------------------------------------------------------
// Alphabet: dense byte <-> symbol map (reference alphabet.hpp:13-47).
class Alphabet {
public:
    static constexpr int16_t kAbsent = -1;

    static Alphabet from_symbols(const uint8_t* symbols, size_t count);
    static Alphabet standard(unsigned sigma);

    unsigned size() const { return unsigned(symbols_.size()); }
    int symbol_of(uint8_t byte) const { return sym_[byte]; }
    bool contains(uint8_t byte) const { return sym_[byte] >= 0; }
    uint8_t byte_of(unsigned symbol) const { return symbols_[symbol]; }
    const std::vector<uint8_t>& symbols() const { return symbols_; }
    const std::array<int16_t, 256>& table() const { return sym_; }
    bool is_identity() const; // sigma 256 in byte order
    bool operator==(const Alphabet& o) const { return symbols_ == o.symbols_; }

private:
    Alphabet() { sym_.fill(kAbsent); }
    std::array<int16_t, 256> sym_{};
    std::vector<uint8_t> symbols_;
};

// ---------------------------------------------------------------------------
// Pattern sets (reference corpus.hpp:27-57, corpus.cpp:12-157).
struct PatternSet {
    std::vector<std::string> patterns; // id = index
    Alphabet alphabet = Alphabet::standard(2);

    static PatternSet create(std::vector<std::string> patterns, Alphabet alphabet);
};

// std::mt19937 is the reference algorithm (624-word state, init_genrand);
// the reference wraps the same engine (corpus.hpp:17-24).
PatternSet generate_patterns(uint32_t seed, const Alphabet& a, uint64_t count, uint32_t length);
void generate_corpus(uint32_t seed, const Alphabet& a, uint64_t bytes, uint8_t* out);
void plant_patterns(uint8_t* corpus, uint64_t bytes, const PatternSet& set, uint64_t occurrences,
                    uint32_t seed);
std::string sha256_hex(const uint8_t* data, uint64_t bytes);
void save_patterns(const PatternSet& set, const std::string& path);
PatternSet load_patterns(const std::string& path, const Alphabet& a, bool hex);

uint32_t minimal_unique_prefix(const std::vector<std::string>& patterns);
uint32_t choose_depth(const PatternSet& set);

// ---------------------------------------------------------------------------
// Canonical trie (reference trie.hpp:45-147).

enum class Stage : uint8_t { None = 0, FinalMerged = 1, TailMerged = 2 };

struct DeviceTrie; // csrc/cuda: per-device image, built lazily on first scan

class Trie {
public:
    static constexpr uint32_t kNone = 0xFFFFFFFFu;
    static constexpr uint32_t kOffsetMask = 0x7FFFFFFFu;
    static constexpr uint32_t kTerminal = 0x80000000u;
    static constexpr uint32_t kMaxNodes = 0x7FFFFFFFu;

    Trie(Alphabet a) : alphabet(std::move(a)), words((alphabet.size() + 31) / 32) {}
    Trie(const Trie&) = delete;
    Trie& operator=(const Trie&) = delete;
    ~Trie();

    Alphabet alphabet;
    uint32_t words;
    uint32_t node_count = 0;
    CellVector cells; // node i: cells[i*stride .. +words) bitmap, then offset word
    std::vector<std::string> patterns;
    uint32_t min_len = 0, max_len = 0;
    Stage stage = Stage::None;
    std::optional<uint32_t> depth_limit;
    // Verification buckets of a truncated trie, ascending by node; ids ascending.
    std::vector<std::pair<uint32_t, std::vector<uint32_t>>> buckets;
    // Read from a .htri file: its language is not known to equal the
    // dictionary, so the GPU image verifies every terminal hit.
    bool loaded = false;

    uint32_t stride() const { return words + 1; }
    const uint32_t* cell(uint32_t n) const { return cells.data() + size_t(n) * stride(); }
    uint32_t offset(uint32_t n) const { return cell(n)[words] & kOffsetMask; }
    bool terminal(uint32_t n) const { return (cell(n)[words] & kTerminal) != 0; }
    uint32_t child_count(uint32_t n) const;
    uint32_t transition(uint32_t node, uint8_t byte) const; // Eq. 1, kNone on miss
    void set_lengths();                                    // min_len / max_len from patterns

    // GPU image, one per device, created on first use (thread-safe).
    std::shared_ptr<DeviceTrie> device_image(int device) const;

private:
    mutable std::mutex dev_mu_;
    mutable std::vector<std::shared_ptr<DeviceTrie>> dev_;
};

struct CompressionStats {
    uint64_t nodes_before = 0, nodes_after_stage1 = 0, nodes_after_stage2 = 0, pattern_count = 0;
    double reduction_percent = 0;
};

double reduction_percent(uint64_t before, uint64_t after);

std::unique_ptr<Trie> build_trie(const PatternSet& set);
std::unique_ptr<Trie> merge_final_nodes(const Trie& t, CompressionStats* stats);
std::unique_ptr<Trie> merge_tail_chains(const Trie& t, CompressionStats* stats);
std::unique_ptr<Trie> truncate_trie(const Trie& t, uint32_t depth, bool* was_noop);
std::vector<uint32_t> first_reach_depths(const Trie& t);
std::vector<std::pair<uint32_t, std::vector<uint32_t>>> verification_buckets(const Trie& t,
                                                                              uint32_t depth);

std::vector<uint8_t> encode_htri(const Trie& t);
std::unique_ptr<Trie> decode_htri(const uint8_t* data, size_t size);
void save_trie(const Trie& t, const std::string& path);
std::unique_ptr<Trie> load_trie(const std::string& path);

std::string format_mib(uint64_t bytes);

} // namespace hfb

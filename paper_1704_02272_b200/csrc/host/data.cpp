// data.cpp -- alphabets, pattern sets, synthetic corpora, pattern files.
//
// Behavioural contract (reference): alphabet.cpp:7-63, corpus.cpp:12-157,
// prefix.cpp:53-100.  Generators must be bit-identical to the reference's
// because callers compare datasets by SHA-256 (acceptance.cpp:274-332).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <random>
#include <unordered_set>

#include "core.hpp"

namespace hfb {

std::string hex_byte(uint8_t b)
{
    static const char* digits = "0123456789abcdef";
    return std::string{digits[b >> 4], digits[b & 15]};
}

// ---- Alphabet ---------------------------------------------------------------

Alphabet Alphabet::from_symbols(const uint8_t* symbols, size_t count)
{
    if (count < 2 || count > 256)
        invalid("alphabet size must be in 2..256, got " + std::to_string(count));
    Alphabet a;
    a.symbols_.assign(symbols, symbols + count);
    for (size_t i = 0; i < count; ++i) {
        uint8_t b = symbols[i];
        if (a.sym_[b] != kAbsent) fail(HEPFAC_ERR_DUPLICATE, "duplicate alphabet byte 0x" + hex_byte(b));
        a.sym_[b] = int16_t(i);
    }
    return a;
}

Alphabet Alphabet::standard(unsigned sigma)
{
    // Canonical orders (reference alphabet.cpp:33-63): DNA for 4, the byte
    // identity for 256, otherwise alphanumerics first, then the remaining
    // printable bytes, then every other byte in ascending order.
    if (sigma == 4) {
        const uint8_t acgt[4] = {'A', 'C', 'G', 'T'};
        return from_symbols(acgt, 4);
    }
    std::vector<uint8_t> order;
    order.reserve(256);
    if (sigma == 256) {
        for (unsigned b = 0; b < 256; ++b) order.push_back(uint8_t(b));
    } else {
        auto alnum = [](unsigned b) {
            return (b >= 'a' && b <= 'z') || (b >= 'A' && b <= 'Z') || (b >= '0' && b <= '9');
        };
        for (unsigned b = 'a'; b <= 'z'; ++b) order.push_back(uint8_t(b));
        for (unsigned b = 'A'; b <= 'Z'; ++b) order.push_back(uint8_t(b));
        for (unsigned b = '0'; b <= '9'; ++b) order.push_back(uint8_t(b));
        for (unsigned b = 33; b < 127; ++b)
            if (!alnum(b)) order.push_back(uint8_t(b));
        for (unsigned b = 0; b < 256; ++b)
            if (b < 33 || b >= 127) order.push_back(uint8_t(b));
    }
    if (sigma < 2 || sigma > order.size())
        invalid("alphabet size must be in 2..256, got " + std::to_string(sigma));
    return from_symbols(order.data(), sigma);
}

bool Alphabet::is_identity() const
{
    if (symbols_.size() != 256) return false;
    for (unsigned i = 0; i < 256; ++i)
        if (symbols_[i] != i) return false;
    return true;
}

// ---- PatternSet -------------------------------------------------------------

PatternSet PatternSet::create(std::vector<std::string> patterns, Alphabet alphabet)
{
    std::unordered_set<std::string_view> seen;
    seen.reserve(patterns.size() * 2);
    for (const auto& p : patterns) {
        if (p.empty()) invalid("empty pattern");
        if (!seen.insert(std::string_view(p)).second) fail(HEPFAC_ERR_DUPLICATE, "duplicate pattern");
        for (unsigned char b : p)
            if (!alphabet.contains(b))
                fail(HEPFAC_ERR_BAD_BYTE, "pattern byte 0x" + hex_byte(b) + " not in alphabet");
    }
    PatternSet s;
    s.patterns = std::move(patterns);
    s.alphabet = std::move(alphabet);
    return s;
}

PatternSet generate_patterns(uint32_t seed, const Alphabet& a, uint64_t count, uint32_t length)
{
    if (count == 0) invalid("pattern count must be >= 1");
    if (length == 0) invalid("pattern length must be >= 1");
    const unsigned sigma = a.size();
    // Feasibility (reference corpus.cpp:39-44): only checked while sigma^length
    // is representable, i.e. below 2^64.
    if (double(length) * std::log2(double(sigma)) < 64.0 &&
        static_cast<long double>(count) > std::pow(static_cast<long double>(sigma), length))
        invalid("cannot generate " + std::to_string(count) + " distinct patterns of length " +
                std::to_string(length) + " over sigma=" + std::to_string(sigma));
    std::mt19937 mt(seed);
    std::unordered_set<std::string> seen;
    seen.reserve(size_t(count) * 2);
    PatternSet s;
    s.alphabet = a;
    s.patterns.reserve(size_t(count));
    std::string draw(length, '\0');
    while (s.patterns.size() < count) {
        for (auto& ch : draw) ch = char(a.byte_of(mt() % sigma));
        if (seen.insert(draw).second) s.patterns.push_back(draw); // rejection of repeats
    }
    return s;
}

void generate_corpus(uint32_t seed, const Alphabet& a, uint64_t bytes, uint8_t* out)
{
    if (bytes == 0) invalid("corpus size must be >= 1");
    std::mt19937 mt(seed);
    const unsigned sigma = a.size();
    for (uint64_t i = 0; i < bytes; ++i) out[i] = a.byte_of(mt() % sigma);
}

void plant_patterns(uint8_t* corpus, uint64_t bytes, const PatternSet& set, uint64_t occurrences,
                    uint32_t seed)
{
    if (set.patterns.empty() || bytes == 0) return;
    std::mt19937 mt(seed);
    const size_t n = set.patterns.size();
    for (uint64_t i = 0; i < occurrences; ++i) {
        const std::string& p = set.patterns[i % n]; // round robin
        if (p.size() > bytes) continue;
        const uint64_t span = bytes - p.size() + 1;
        // The reference draws the two 32-bit halves inside one expression
        // (corpus.cpp:81); its g++ build evaluates the high half first.
        // tests/test_host_parity.py pins this order against the compiled reference.
        const uint64_t hi = mt();
        const uint64_t lo = mt();
        const uint64_t at = ((hi << 32) | lo) % span;
        std::memcpy(corpus + at, p.data(), p.size());
    }
}

// ---- SHA-256 (FIPS 180-4), self-contained -------------------------------------

namespace {
struct Sha256 {
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                     0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
    void block(const uint8_t* p)
    {
        static const uint32_t k[64] = {
            0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
            0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
            0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
            0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
            0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
            0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
            0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
            0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
            0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
            0xc67178f2};
        uint32_t w[64];
        for (int i = 0; i < 16; ++i)
            w[i] = uint32_t(p[4 * i]) << 24 | uint32_t(p[4 * i + 1]) << 16 |
                   uint32_t(p[4 * i + 2]) << 8 | p[4 * i + 3];
        for (int i = 16; i < 64; ++i) {
            uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
            uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
            w[i] = w[i - 16] + s0 + w[i - 7] + s1;
        }
        uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
        for (int i = 0; i < 64; ++i) {
            uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + k[i] + w[i];
            uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
            hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
    }
};
} // namespace

std::string sha256_hex(const uint8_t* data, uint64_t bytes)
{
    Sha256 s;
    uint64_t full = bytes / 64;
    for (uint64_t i = 0; i < full; ++i) s.block(data + 64 * i);
    uint8_t tail[128] = {0};
    uint64_t rem = bytes - full * 64;
    if (rem) std::memcpy(tail, data + full * 64, size_t(rem));
    tail[rem] = 0x80;
    size_t tail_len = rem + 1 + 8 <= 64 ? 64 : 128;
    uint64_t bits = bytes * 8;
    for (int i = 0; i < 8; ++i) tail[tail_len - 1 - i] = uint8_t(bits >> (8 * i));
    s.block(tail);
    if (tail_len == 128) s.block(tail + 64);
    std::string out;
    for (uint32_t v : s.h)
        for (int sh = 24; sh >= 0; sh -= 8) out += hex_byte(uint8_t(v >> sh));
    return out;
}

// ---- pattern files (reference corpus.cpp:109-157) ---------------------------

void save_patterns(const PatternSet& set, const std::string& path)
{
    std::ofstream f(path, std::ios::binary);
    if (!f) fail(HEPFAC_ERR_IO, "cannot open " + path + " for writing");
    const bool hex = set.alphabet.contains(uint8_t('\n')); // raw lines would be ambiguous
    std::string buf;
    for (const auto& p : set.patterns) {
        if (hex)
            for (unsigned char b : p) buf += hex_byte(b);
        else
            buf += p;
        buf += '\n';
    }
    f.write(buf.data(), std::streamsize(buf.size()));
    if (!f) fail(HEPFAC_ERR_IO, "write failed: " + path);
}

PatternSet load_patterns(const std::string& path, const Alphabet& a, bool hex)
{
    std::ifstream f(path, std::ios::binary);
    if (!f) fail(HEPFAC_ERR_IO, "cannot open " + path);
    std::string content((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    auto nibble = [&](char c) -> unsigned {
        if (c >= '0' && c <= '9') return unsigned(c - '0');
        if (c >= 'a' && c <= 'f') return unsigned(c - 'a' + 10);
        if (c >= 'A' && c <= 'F') return unsigned(c - 'A' + 10);
        fail(HEPFAC_ERR_INTERNAL, "invalid hex digit in " + path);
    };
    std::vector<std::string> out;
    size_t pos = 0;
    while (pos < content.size()) {
        size_t nl = content.find('\n', pos);
        size_t end = nl == std::string::npos ? content.size() : nl;
        std::string_view line(content.data() + pos, end - pos);
        pos = nl == std::string::npos ? content.size() : nl + 1;
        if (line.empty()) continue;
        if (!hex) {
            out.emplace_back(line);
            continue;
        }
        if (line.size() % 2) fail(HEPFAC_ERR_INTERNAL, "odd-length hex pattern line in " + path);
        std::string raw(line.size() / 2, '\0');
        for (size_t i = 0; i < raw.size(); ++i)
            raw[i] = char((nibble(line[2 * i]) << 4) | nibble(line[2 * i + 1]));
        out.push_back(std::move(raw));
    }
    return PatternSet::create(std::move(out), a);
}

// ---- prefix policy (reference prefix.cpp:53-73, 94-100) -----------------------

uint32_t minimal_unique_prefix(const std::vector<std::string>& patterns)
{
    // Truncations p[:min(d,|p|)] collide for a pair exactly when d <= LCP(p, q),
    // so the answer is max(1, 1 + longest common prefix of any pair), and the
    // longest pairwise LCP is attained between lexicographic neighbours.
    if (patterns.empty()) invalid("empty pattern set");
    std::vector<std::string_view> v(patterns.begin(), patterns.end());
    std::sort(v.begin(), v.end());
    uint32_t best = 1;
    for (size_t i = 1; i < v.size(); ++i) {
        if (v[i] == v[i - 1]) fail(HEPFAC_ERR_DUPLICATE, "pattern set contains duplicates");
        size_t n = std::min(v[i].size(), v[i - 1].size()), l = 0;
        while (l < n && v[i][l] == v[i - 1][l]) ++l;
        best = std::max<uint32_t>(best, uint32_t(l + 1));
    }
    return best;
}

uint32_t choose_depth(const PatternSet& set)
{
    uint32_t shortest = UINT32_MAX;
    for (const auto& p : set.patterns) shortest = std::min<uint32_t>(shortest, uint32_t(p.size()));
    uint32_t d = set.alphabet.size() > 52 ? 5u : minimal_unique_prefix(set.patterns);
    return std::max<uint32_t>(1, std::min(d, shortest));
}

} // namespace hfb

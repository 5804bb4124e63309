// htri.cpp -- the .htri trie file (reference trie_io.hpp:13-27,
// trie_io.cpp:64-166).  Little-endian:
//   "HTRI" u16 version=1, u16 sigma, u32 node_count, u16 words
//   node_count*(words+1) u32 cells
//   u32 n; n x { u16 len, len bytes, u32 id }
//   "HTRX" u16 version=1, u8 stage, u8 has_limit, u16 limit, u16 alen, alen bytes
// A file without the HTRX trailer is a stage-0 trie over standard(sigma).
#include <cstring>
#include <fstream>
#include <iterator>

#include "core.hpp"

namespace hfb {

namespace {

struct Writer {
    std::vector<uint8_t> b;
    void u8(uint8_t x) { b.push_back(x); }
    void u16(uint16_t x) { u8(uint8_t(x)), u8(uint8_t(x >> 8)); }
    void u32(uint32_t x) { u16(uint16_t(x)), u16(uint16_t(x >> 16)); }
    void raw(const void* p, size_t n)
    {
        auto* c = static_cast<const uint8_t*>(p);
        b.insert(b.end(), c, c + n);
    }
};

struct Cursor {
    const uint8_t* p;
    size_t size, at = 0;
    size_t left() const { return size - at; }
    void need(size_t n) const
    {
        if (n > left()) fail(HEPFAC_ERR_FORMAT, "trie file truncated");
    }
    uint8_t u8() { return need(1), p[at++]; }
    uint16_t u16()
    {
        need(2);
        uint16_t x = uint16_t(p[at] | (p[at + 1] << 8));
        at += 2;
        return x;
    }
    uint32_t u32()
    {
        uint32_t lo = u16();
        return lo | (uint32_t(u16()) << 16);
    }
    bool tag(const char* t)
    {
        if (left() < 4 || std::memcmp(p + at, t, 4) != 0) return false;
        at += 4;
        return true;
    }
};

} // namespace

std::vector<uint8_t> encode_htri(const Trie& t)
{
    Writer w;
    w.b.reserve(32 + t.cells.size() * 4);
    w.raw("HTRI", 4);
    w.u16(1);
    w.u16(uint16_t(t.alphabet.size()));
    w.u32(t.node_count);
    w.u16(uint16_t(t.words));
    for (uint32_t c : t.cells) w.u32(c);
    w.u32(uint32_t(t.patterns.size()));
    for (uint32_t id = 0; id < t.patterns.size(); ++id) {
        w.u16(uint16_t(t.patterns[id].size()));
        w.raw(t.patterns[id].data(), t.patterns[id].size());
        w.u32(id);
    }
    w.raw("HTRX", 4);
    w.u16(1);
    w.u8(uint8_t(t.stage));
    w.u8(t.depth_limit ? 1 : 0);
    w.u16(uint16_t(t.depth_limit.value_or(0)));
    w.u16(uint16_t(t.alphabet.size()));
    w.raw(t.alphabet.symbols().data(), t.alphabet.size());
    return std::move(w.b);
}

std::unique_ptr<Trie> decode_htri(const uint8_t* data, size_t size)
{
    Cursor r{data, size};
    if (!r.tag("HTRI")) fail(HEPFAC_ERR_FORMAT, "not a trie file (bad magic)");
    if (r.u16() != 1) fail(HEPFAC_ERR_FORMAT, "unsupported trie format version");
    uint32_t sigma = r.u16();
    if (sigma == 0) sigma = 256;
    if (sigma < 2 || sigma > 256) fail(HEPFAC_ERR_FORMAT, "invalid sigma in trie file");
    const uint32_t nodes = r.u32();
    const uint32_t words = r.u16();
    if (words != (sigma + 31) / 32) fail(HEPFAC_ERR_FORMAT, "bitmap width mismatch");
    if (nodes == 0 || nodes > Trie::kMaxNodes) fail(HEPFAC_ERR_INTERNAL, "invalid node count");

    const size_t ncells = size_t(nodes) * (words + 1);
    r.need(ncells * 4);
    CellVector cells(ncells);
    for (auto& c : cells) c = r.u32();

    const uint32_t count = r.u32();
    r.need(size_t(count) * 6);
    std::vector<std::string> patterns(count);
    std::vector<uint8_t> seen(count, 0);
    for (uint32_t i = 0; i < count; ++i) {
        const uint16_t len = r.u16();
        r.need(len);
        std::string p(reinterpret_cast<const char*>(r.p + r.at), len);
        r.at += len;
        const uint32_t id = r.u32();
        if (id >= count || seen[id]) fail(HEPFAC_ERR_INTERNAL, "invalid pattern id");
        seen[id] = 1;
        patterns[id] = std::move(p);
    }

    Stage stage = Stage::None;
    std::optional<uint32_t> limit;
    std::optional<Alphabet> alphabet;
    if (r.left() > 0 && r.tag("HTRX")) {
        if (r.u16() != 1) fail(HEPFAC_ERR_INTERNAL, "unsupported trie trailer version");
        const uint8_t st = r.u8();
        if (st > 2) fail(HEPFAC_ERR_INTERNAL, "invalid compression stage");
        stage = Stage(st);
        const uint8_t has_limit = r.u8();
        const uint16_t lim = r.u16();
        if (has_limit) limit = lim;
        const uint16_t alen = r.u16();
        r.need(alen);
        alphabet = Alphabet::from_symbols(r.p + r.at, alen);
        r.at += alen;
        if (alphabet->size() != sigma) fail(HEPFAC_ERR_FORMAT, "alphabet/sigma mismatch");
    } else {
        alphabet = Alphabet::standard(sigma);
    }

    for (uint32_t n = 0; n < nodes; ++n) {
        const uint32_t off = cells[size_t(n) * (words + 1) + words] & Trie::kOffsetMask;
        if (off != 0 && off >= nodes) fail(HEPFAC_ERR_INTERNAL, "offset out of range");
    }

    auto t = std::make_unique<Trie>(std::move(*alphabet));
    t->node_count = nodes;
    t->cells = std::move(cells);
    t->patterns = std::move(patterns);
    t->set_lengths();
    t->stage = stage;
    t->depth_limit = limit;
    t->loaded = true;
    if (limit) t->buckets = verification_buckets(*t, *limit);
    return t;
}

void save_trie(const Trie& t, const std::string& path)
{
    const auto bytes = encode_htri(t);
    std::ofstream f(path, std::ios::binary);
    if (!f) fail(HEPFAC_ERR_IO, "cannot open " + path + " for writing");
    f.write(reinterpret_cast<const char*>(bytes.data()), std::streamsize(bytes.size()));
    if (!f) fail(HEPFAC_ERR_IO, "write failed: " + path);
}

std::unique_ptr<Trie> load_trie(const std::string& path)
{
    std::ifstream f(path, std::ios::binary);
    if (!f) fail(HEPFAC_ERR_IO, "cannot open " + path);
    std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (f.bad()) fail(HEPFAC_ERR_IO, "read failed: " + path);
    return decode_htri(bytes.data(), bytes.size());
}

} // namespace hfb

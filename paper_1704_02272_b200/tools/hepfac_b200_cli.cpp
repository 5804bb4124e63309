// hepfac_b200_cli -- command-line front end of the B200 library, covering the
// reference CLI's end-to-end user path (reference tools/hepfac_cli.cpp):
//
//   build --patterns FILE [--sigma N] [--hex] [--compress 0|1|2] [--out TRIE]
//         pattern file -> .htri, JSON report (compression stats, memory) on stdout
//   match --trie TRIE --input FILE [--workers N] [--chunk N] [--depth D] [--out FILE]
//         "start\tlength\tid" lines (stdout or --out), JSON timing summary on stderr
//
// Defaults, report fields and exit codes follow the reference (sigma 52,
// compress 0, out trie.htri; exit 0 ok, 1 invalid input, 2 I/O or format).
// The match lines are byte-identical to the reference's for the same trie and
// input.  Everything goes through the public C ABI (hepfac.h).
//
// Design: options are declared once in a table (name, takes-value) and parsed
// into a map; handles are unique_ptrs with the ABI's destroy functions as
// deleters; the input file is memory-mapped, so the text reaches hepfac_scan
// as a pageable borrowed pointer (staged by the library's pinned ring) without
// a read copy; output lines are formatted into one buffer and written once.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cinttypes>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "hepfac.h"

namespace {

enum Exit : int { kOk = 0, kInvalid = 1, kIo = 2 };

// Error path: message to stderr, process exit code from the status class.
struct CliError {
    int code;
    std::string message;
};

Exit exit_class(hepfac_status_t s)
{
    switch (s) {
    case HEPFAC_OK: return kOk;
    case HEPFAC_ERR_IO:
    case HEPFAC_ERR_FORMAT: return kIo;
    default: return kInvalid;
    }
}

void ok_or_throw(hepfac_status_t s, const char* what)
{
    if (s == HEPFAC_OK) return;
    std::string m = std::string(what) + ": " + hepfac_status_string(s);
    const char* detail = hepfac_last_error();
    if (detail && detail[0]) m += std::string(" (") + detail + ")";
    throw CliError{exit_class(s), m};
}

constexpr const char* kUsage =
    "usage:\n"
    "  hepfac_b200_cli build --patterns FILE [--sigma N] [--hex] [--compress 0|1|2] [--out TRIE]\n"
    "  hepfac_b200_cli match --trie TRIE --input FILE [--workers N] [--chunk N] [--depth D] [--out FILE]\n";

[[noreturn]] void bad_usage(const std::string& why) { throw CliError{kInvalid, why + "\n" + kUsage}; }

// ---- options ---------------------------------------------------------------

struct OptionSpec {
    const char* name;
    bool value;
};

class Options {
public:
    Options(int argc, char** argv, std::initializer_list<OptionSpec> spec)
    {
        for (int i = 2; i < argc; ++i) {
            const std::string tok = argv[i];
            const OptionSpec* hit = nullptr;
            for (const auto& s : spec)
                if (tok == s.name) hit = &s;
            if (!hit) bad_usage("unknown argument " + tok);
            if (!hit->value) {
                values_[tok] = "";
                continue;
            }
            if (i + 1 == argc) bad_usage(tok + " needs a value");
            values_[tok] = argv[++i];
        }
    }
    bool has(const std::string& k) const { return values_.count(k) != 0; }
    std::string text(const std::string& k, const std::string& fallback = "") const
    {
        auto it = values_.find(k);
        return it == values_.end() ? fallback : it->second;
    }
    uint64_t number(const std::string& k, uint64_t fallback) const
    {
        auto it = values_.find(k);
        if (it == values_.end()) return fallback;
        const std::string& v = it->second;
        uint64_t x = 0;
        if (v.empty()) bad_usage(k + " must be a non-negative integer");
        for (char c : v) {
            if (c < '0' || c > '9') bad_usage(k + " must be a non-negative integer");
            x = x * 10 + uint64_t(c - '0');
        }
        return x;
    }

private:
    std::map<std::string, std::string> values_;
};

// ---- handles -----------------------------------------------------------------

using AlphabetPtr = std::unique_ptr<hepfac_alphabet_t, decltype(&hepfac_alphabet_destroy)>;
using PatternsPtr = std::unique_ptr<hepfac_patterns_t, decltype(&hepfac_patterns_destroy)>;
using TriePtr = std::unique_ptr<hepfac_trie_t, decltype(&hepfac_trie_destroy)>;
using ListPtr = std::unique_ptr<hepfac_match_list_t, decltype(&hepfac_match_list_destroy)>;

TriePtr no_trie() { return TriePtr(nullptr, &hepfac_trie_destroy); }

// ---- files -------------------------------------------------------------------

// Read-only mapping of a whole file (an empty file maps to nothing).
class MappedFile {
public:
    explicit MappedFile(const std::string& path)
    {
        fd_ = ::open(path.c_str(), O_RDONLY);
        if (fd_ < 0) throw CliError{kIo, "cannot open " + path};
        struct stat st {};
        if (::fstat(fd_, &st) != 0) throw CliError{kIo, "cannot stat " + path};
        size_ = size_t(st.st_size);
        if (size_) {
            void* p = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd_, 0);
            if (p == MAP_FAILED) throw CliError{kIo, "cannot map " + path};
            data_ = static_cast<const uint8_t*>(p);
        }
    }
    ~MappedFile()
    {
        if (data_) ::munmap(const_cast<uint8_t*>(data_), size_);
        if (fd_ >= 0) ::close(fd_);
    }
    MappedFile(const MappedFile&) = delete;
    const uint8_t* data() const { return data_; }
    size_t size() const { return size_; }

private:
    int fd_ = -1;
    const uint8_t* data_ = nullptr;
    size_t size_ = 0;
};

void write_all(FILE* f, const std::string& bytes, const std::string& what)
{
    if (!bytes.empty() && std::fwrite(bytes.data(), 1, bytes.size(), f) != bytes.size())
        throw CliError{kIo, "write failed: " + what};
}

// ---- JSON (the two small reports) ---------------------------------------------

// Pretty: one key per line, two spaces per level (the build report);
// compact: one line (the match summary).
class Json {
public:
    explicit Json(bool pretty) : pretty_(pretty) {}
    Json& open() { return raw("{"), first_ = true, *this; }
    Json& close(int indent) { return newline(indent - 2), raw("}"), first_ = false, *this; }
    Json& key(const char* k, int indent)
    {
        if (!first_) raw(",");
        first_ = false;
        newline(indent);
        return raw("\""), raw(k), raw(pretty_ ? "\": " : "\":");
    }
    Json& num(uint64_t v) { return raw(std::to_string(v)); }
    Json& real(double v)
    {
        char b[40];
        std::snprintf(b, sizeof b, "%.17g", v);
        return raw(b);
    }
    Json& str(const std::string& s)
    {
        raw("\"");
        for (char c : s) {
            if (c == '"' || c == '\\') out_ += '\\';
            out_ += c;
        }
        return raw("\"");
    }
    const std::string& text() const { return out_; }

private:
    Json& raw(const std::string& s) { return out_ += s, *this; }
    void newline(int indent)
    {
        if (pretty_) out_ += "\n" + std::string(size_t(indent), ' ');
    }
    std::string out_;
    bool pretty_;
    bool first_ = true;
};

// ---- subcommands ---------------------------------------------------------------

int run_build(const Options& o)
{
    if (!o.has("--patterns")) bad_usage("build: --patterns is required");
    const std::string out = o.text("--out", "trie.htri");
    const uint64_t sigma = o.number("--sigma", 52);
    const uint64_t stages = o.number("--compress", 0);
    if (stages > 2) bad_usage("--compress must be 0, 1 or 2");

    hepfac_alphabet_t* a = nullptr;
    ok_or_throw(hepfac_alphabet_standard(uint16_t(sigma), &a), "alphabet");
    AlphabetPtr alphabet(a, &hepfac_alphabet_destroy);
    hepfac_patterns_t* p = nullptr;
    ok_or_throw(hepfac_patterns_load(o.text("--patterns").c_str(), alphabet.get(), o.has("--hex") ? 1 : 0, &p),
                "pattern file");
    PatternsPtr patterns(p, &hepfac_patterns_destroy);
    hepfac_trie_t* t = nullptr;
    ok_or_throw(hepfac_trie_build(patterns.get(), &t), "trie build");
    TriePtr trie(t, &hepfac_trie_destroy);

    Json j(true);
    j.open();
    if (stages) {
        hepfac_compression_stats_t cs{};
        hepfac_trie_t* c = nullptr;
        ok_or_throw(hepfac_trie_compress_stats(trie.get(), int(stages), &c, &cs), "compression");
        trie.reset(c);
        j.key("compression", 2).open();
        j.key("nodes_before", 4).num(cs.nodes_before);
        j.key("nodes_after_stage1", 4).num(cs.nodes_after_stage1);
        j.key("nodes_after_stage2", 4).num(cs.nodes_after_stage2);
        j.key("pattern_count", 4).num(cs.pattern_count);
        j.key("reduction_percent", 4).real(cs.reduction_percent);
        j.close(4);
    }
    ok_or_throw(hepfac_trie_save(trie.get(), out.c_str()), "trie save");
    hepfac_memory_report_t mem{};
    ok_or_throw(hepfac_trie_memory_report(trie.get(), &mem), "memory report");
    j.key("memory", 2).open();
    j.key("node_count", 4).num(mem.node_count);
    j.key("bytes_per_node", 4).num(mem.bytes_per_node);
    j.key("total_bytes", 4).num(mem.total_bytes);
    j.key("total_mib", 4).str(mem.total_mib);
    j.key("sigma", 4).num(mem.sigma);
    j.close(4);
    j.key("trie", 2).str(out);
    j.close(2);
    write_all(stdout, j.text() + "\n", "stdout");
    return kOk;
}

int run_match(const Options& o)
{
    if (!o.has("--trie") || !o.has("--input")) bad_usage("match: --trie and --input are required");
    uint64_t workers = o.number("--workers", 0);
    if (!o.has("--workers"))
        if (const char* env = std::getenv("HEPFAC_WORKERS")) workers = std::strtoull(env, nullptr, 10);
    const hepfac_scan_config_t config{uint32_t(workers), uint32_t(o.number("--chunk", 0))};
    const uint64_t depth = o.number("--depth", 0);

    hepfac_trie_t* t = nullptr;
    ok_or_throw(hepfac_trie_load(o.text("--trie").c_str(), &t), "trie load");
    TriePtr trie(t, &hepfac_trie_destroy), truncated = no_trie();
    if (depth) {
        hepfac_trie_t* d = nullptr;
        int noop = 0;
        ok_or_throw(hepfac_trie_truncate(trie.get(), uint32_t(depth), &d, &noop), "truncate");
        truncated.reset(d);
    }
    const hepfac_trie_t* active = truncated ? truncated.get() : trie.get();
    const MappedFile input(o.text("--input"));

    // one timed run first (the reference reports run_throughput's figures;
    // it refuses an empty corpus, so an empty input reports zeros)
    hepfac_throughput_report_t rep{};
    if (input.size())
        ok_or_throw(hepfac_run_throughput(active, input.data(), input.size(), &config, 1, &rep), "throughput");
    hepfac_match_list_t* l = nullptr;
    ok_or_throw(hepfac_scan(active, input.data(), input.size(), &config, &l), "scan");
    const ListPtr list(l, &hepfac_match_list_destroy);

    const size_t n = hepfac_match_list_size(list.get());
    const hepfac_match_t* m = hepfac_match_list_data(list.get());
    std::string lines;
    lines.resize(n * 43 + 1); // u64 (20 digits) + two u32 (10), two tabs, newline; + sprintf's NUL
    char* w = lines.data();
    for (size_t i = 0; i < n; ++i)
        w += std::sprintf(w, "%" PRIu64 "\t%" PRIu32 "\t%" PRIu32 "\n", m[i].start, m[i].length, m[i].pattern_id);
    lines.resize(size_t(w - lines.data()));
    if (o.has("--out")) {
        const std::string path = o.text("--out");
        FILE* f = std::fopen(path.c_str(), "wb");
        if (!f) throw CliError{kIo, "cannot open " + path};
        const std::unique_ptr<FILE, int (*)(FILE*)> closer(f, &std::fclose);
        write_all(f, lines, path);
    } else {
        write_all(stdout, lines, "stdout");
    }
    // timing on stderr, so the match lines stay byte-identical across runs
    Json j(false);
    j.open();
    j.key("matches", 0).num(n);
    j.key("bytes", 0).num(rep.bytes);
    j.key("seconds", 0).real(rep.seconds);
    j.key("gbps", 0).real(rep.gbps);
    j.key("workers", 0).num(rep.workers);
    j.close(2);
    std::fprintf(stderr, "%s\n", j.text().c_str());
    return kOk;
}

} // namespace

int main(int argc, char** argv)
{
    try {
        if (argc < 2) bad_usage("missing subcommand");
        const std::string sub = argv[1];
        if (sub == "build")
            return run_build(Options(argc, argv, {{"--patterns", true},
                                                  {"--sigma", true},
                                                  {"--compress", true},
                                                  {"--out", true},
                                                  {"--hex", false}}));
        if (sub == "match")
            return run_match(Options(argc, argv, {{"--trie", true},
                                                  {"--input", true},
                                                  {"--workers", true},
                                                  {"--chunk", true},
                                                  {"--depth", true},
                                                  {"--out", true}}));
        bad_usage("unknown subcommand " + sub);
    } catch (const CliError& e) {
        std::fprintf(stderr, "hepfac: %s\n", e.message.c_str());
        return e.code;
    }
}

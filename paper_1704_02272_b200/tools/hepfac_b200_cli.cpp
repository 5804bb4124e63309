// hepfac_b200_cli -- the reference CLI's end-to-end user path over the B200
// library: `build` (pattern file -> .htri) and `match` (.htri + input file ->
// match lines), with the reference's arguments, output formats and exit codes
// (reference tools/hepfac_cli.cpp:156-193 cmd_build, :234-279 cmd_match,
// :21-45 exit codes).  Like the reference it talks to the engine only through
// hepfac.h; the argument parser is hand-written (the reference's CLI11 is not
// vendored).
//
//   hepfac_b200_cli build --patterns FILE [--sigma N (52)] [--hex] [--compress 0|1|2 (0)] [--out TRIE]
//   hepfac_b200_cli match --trie TRIE --input FILE [--workers N] [--chunk N] [--depth D] [--out FILE]
//
// `match` writes "start\tlength\tid" lines to stdout (or --out) and a JSON
// summary {matches, bytes, seconds, gbps, workers} to stderr.  The lines are
// byte-identical to the reference's for the same trie and input.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <string>
#include <vector>

#include "hepfac.h"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitValidation = 1;
constexpr int kExitIo = 2;

int exit_code_for(hepfac_status_t s)
{
    if (s == HEPFAC_OK) return kExitOk;
    if (s == HEPFAC_ERR_IO || s == HEPFAC_ERR_FORMAT) return kExitIo;
    return kExitValidation;
}

[[noreturn]] void fail(hepfac_status_t s, const std::string& context)
{
    std::cerr << "hepfac: " << context << ": " << hepfac_status_string(s);
    const char* detail = hepfac_last_error();
    if (detail && *detail) std::cerr << " (" << detail << ")";
    std::cerr << "\n";
    std::exit(exit_code_for(s));
}

void check(hepfac_status_t s, const std::string& context)
{
    if (s != HEPFAC_OK) fail(s, context);
}

[[noreturn]] void usage(const std::string& why)
{
    if (!why.empty()) std::cerr << "hepfac: " << why << "\n";
    std::cerr << "usage:\n"
                 "  hepfac_b200_cli build --patterns FILE [--sigma N] [--hex] [--compress 0|1|2] [--out TRIE]\n"
                 "  hepfac_b200_cli match --trie TRIE --input FILE [--workers N] [--chunk N] [--depth D] "
                 "[--out FILE]\n";
    std::exit(kExitValidation);
}

struct AlphabetHandle {
    hepfac_alphabet_t* ptr = nullptr;
    ~AlphabetHandle() { hepfac_alphabet_destroy(ptr); }
};
struct PatternsHandle {
    hepfac_patterns_t* ptr = nullptr;
    ~PatternsHandle() { hepfac_patterns_destroy(ptr); }
};
struct TrieHandle {
    hepfac_trie_t* ptr = nullptr;
    ~TrieHandle() { hepfac_trie_destroy(ptr); }
};

std::vector<uint8_t> read_file(const std::string& path)
{
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) {
        std::cerr << "hepfac: cannot open " << path << "\n";
        std::exit(kExitIo);
    }
    std::vector<uint8_t> data(size_t(f.tellg()));
    f.seekg(0);
    f.read(reinterpret_cast<char*>(data.data()), std::streamsize(data.size()));
    if (!f) {
        std::cerr << "hepfac: read failed: " << path << "\n";
        std::exit(kExitIo);
    }
    return data;
}

void write_file(const std::string& path, const void* data, size_t size)
{
    std::ofstream f(path, std::ios::binary);
    if (!f || !f.write(static_cast<const char*>(data), std::streamsize(size))) {
        std::cerr << "hepfac: write failed: " << path << "\n";
        std::exit(kExitIo);
    }
}

uint32_t env_workers()
{
    if (const char* env = std::getenv("HEPFAC_WORKERS")) {
        long v = std::strtol(env, nullptr, 10);
        if (v >= 1) return uint32_t(v);
    }
    return 0;
}

// --name value pairs and --flags after the subcommand
struct Args {
    std::vector<std::pair<std::string, std::string>> kv;
    std::vector<std::string> flags;
    bool has(const std::string& k) const
    {
        for (auto& p : kv)
            if (p.first == k) return true;
        return false;
    }
    std::string get(const std::string& k, const std::string& def = "") const
    {
        for (auto& p : kv)
            if (p.first == k) return p.second;
        return def;
    }
    bool flag(const std::string& k) const
    {
        for (auto& f : flags)
            if (f == k) return true;
        return false;
    }
};

Args parse(int argc, char** argv, const std::vector<std::string>& options, const std::vector<std::string>& flag_names)
{
    Args a;
    for (int i = 2; i < argc; ++i) {
        const std::string s = argv[i];
        bool known = false;
        for (auto& f : flag_names)
            if (s == f) a.flags.push_back(s), known = true;
        if (known) continue;
        for (auto& o : options)
            if (s == o) {
                if (i + 1 >= argc) usage(s + " needs a value");
                a.kv.emplace_back(s, argv[++i]);
                known = true;
            }
        if (!known) usage("unknown argument " + s);
    }
    return a;
}

uint64_t to_u64(const std::string& s, const std::string& name)
{
    char* end = nullptr;
    const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
    if (s.empty() || *end) usage(name + " must be a non-negative integer");
    return v;
}

std::string jnum(double v)
{
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

std::string jstr(const std::string& s)
{
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

int cmd_build(const Args& a)
{
    if (!a.has("--patterns")) usage("build: --patterns is required");
    const std::string out_path = a.get("--out", "trie.htri");
    const uint64_t sigma = to_u64(a.get("--sigma", "52"), "--sigma"); // the reference's defaults
    const uint64_t stages = to_u64(a.get("--compress", "0"), "--compress");
    if (stages > 2) usage("--compress must be 0, 1 or 2");
    AlphabetHandle alphabet;
    check(hepfac_alphabet_standard(uint16_t(sigma), &alphabet.ptr), "alphabet");
    PatternsHandle patterns;
    check(hepfac_patterns_load(a.get("--patterns").c_str(), alphabet.ptr, a.flag("--hex") ? 1 : 0, &patterns.ptr),
          "pattern file");
    TrieHandle trie;
    check(hepfac_trie_build(patterns.ptr, &trie.ptr), "trie build");
    std::string report = "{\n";
    TrieHandle compressed;
    const hepfac_trie_t* final_trie = trie.ptr;
    if (stages > 0) {
        hepfac_compression_stats_t st{};
        check(hepfac_trie_compress_stats(trie.ptr, int(stages), &compressed.ptr, &st), "compression");
        final_trie = compressed.ptr;
        report += "  \"compression\": {\n    \"nodes_before\": " + std::to_string(st.nodes_before) +
                  ",\n    \"nodes_after_stage1\": " + std::to_string(st.nodes_after_stage1) +
                  ",\n    \"nodes_after_stage2\": " + std::to_string(st.nodes_after_stage2) +
                  ",\n    \"pattern_count\": " + std::to_string(st.pattern_count) +
                  ",\n    \"reduction_percent\": " + jnum(st.reduction_percent) + "\n  },\n";
    }
    check(hepfac_trie_save(final_trie, out_path.c_str()), "trie save");
    hepfac_memory_report_t mem{};
    check(hepfac_trie_memory_report(final_trie, &mem), "memory report");
    report += "  \"memory\": {\n    \"node_count\": " + std::to_string(mem.node_count) +
              ",\n    \"bytes_per_node\": " + std::to_string(mem.bytes_per_node) +
              ",\n    \"total_bytes\": " + std::to_string(mem.total_bytes) + ",\n    \"total_mib\": " +
              jstr(mem.total_mib) + ",\n    \"sigma\": " + std::to_string(mem.sigma) + "\n  },\n  \"trie\": " +
              jstr(out_path) + "\n}\n";
    std::cout << report;
    return kExitOk;
}

int cmd_match(const Args& a)
{
    if (!a.has("--trie") || !a.has("--input")) usage("match: --trie and --input are required");
    const uint32_t workers = a.has("--workers") ? uint32_t(to_u64(a.get("--workers"), "--workers")) : env_workers();
    const uint32_t chunk = uint32_t(to_u64(a.get("--chunk", "0"), "--chunk"));
    const uint32_t depth = uint32_t(to_u64(a.get("--depth", "0"), "--depth"));
    TrieHandle loaded;
    check(hepfac_trie_load(a.get("--trie").c_str(), &loaded.ptr), "trie load");
    TrieHandle truncated;
    const hepfac_trie_t* trie = loaded.ptr;
    if (depth > 0) {
        int noop = 0;
        check(hepfac_trie_truncate(loaded.ptr, depth, &truncated.ptr, &noop), "truncate");
        trie = truncated.ptr;
    }
    std::vector<uint8_t> text = read_file(a.get("--input"));
    hepfac_scan_config_t config{workers, chunk};

    hepfac_throughput_report_t rep{};
    if (!text.empty()) // the reference's run_throughput refuses an empty corpus
        check(hepfac_run_throughput(trie, text.data(), text.size(), &config, 1, &rep), "throughput");

    hepfac_match_list_t* list = nullptr;
    check(hepfac_scan(trie, text.data(), text.size(), &config, &list), "scan");
    std::unique_ptr<hepfac_match_list_t, decltype(&hepfac_match_list_destroy)> guard(list,
                                                                                      &hepfac_match_list_destroy);
    const hepfac_match_t* data = hepfac_match_list_data(list);
    const size_t n = hepfac_match_list_size(list);
    std::string lines;
    lines.reserve(n * 24);
    char buf[96];
    for (size_t i = 0; i < n; ++i) {
        const int k = std::snprintf(buf, sizeof buf, "%llu\t%u\t%u\n", (unsigned long long)data[i].start,
                                    data[i].length, data[i].pattern_id);
        lines.append(buf, size_t(k));
    }
    if (a.has("--out")) write_file(a.get("--out"), lines.data(), lines.size());
    else std::cout << lines;
    // timing goes to stderr so the match list stays byte-identical across runs
    std::cerr << "{\"matches\":" << n << ",\"bytes\":" << rep.bytes << ",\"seconds\":" << jnum(rep.seconds)
              << ",\"gbps\":" << jnum(rep.gbps) << ",\"workers\":" << rep.workers << "}\n";
    return kExitOk;
}

} // namespace

int main(int argc, char** argv)
{
    if (argc < 2) usage("");
    const std::string cmd = argv[1];
    if (cmd == "build") return cmd_build(parse(argc, argv, {"--patterns", "--sigma", "--compress", "--out"}, {"--hex"}));
    if (cmd == "match")
        return cmd_match(parse(argc, argv, {"--trie", "--input", "--workers", "--chunk", "--depth", "--out"}, {}));
    usage("unknown subcommand " + cmd);
}

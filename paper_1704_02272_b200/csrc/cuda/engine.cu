// engine.cu -- host runtime of the GPU match engine: device images of tries,
// pooled per-call workspaces (stream, buffers, tile status), the streaming
// H2D -> kernel -> D2H pipeline behind hepfac_scan, run_throughput and the
// device-resident benchmark session.  No CPU fallback: without a usable
// sm_100a device every entry point fails with HEPFAC_ERR_INTERNAL.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "../host/image.hpp"
#include "engine.hpp"
#include "dna_kernel.cuh"
#include "filter_kernel.cuh"
#include "scan_kernel.cuh"

namespace hfb {

// ---------------------------------------------------------------------------
// errors

namespace {

[[noreturn]] void cuda_fail(cudaError_t e, const char* what)
{
    const hepfac_status_t s = e == cudaErrorMemoryAllocation ? HEPFAC_ERR_NOMEM : HEPFAC_ERR_INTERNAL;
    fail(s, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

#define CK(x)                                      \
    do {                                           \
        cudaError_t e_ = (x);                      \
        if (e_ != cudaSuccess) cuda_fail(e_, #x);  \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d)
    {
        cudaGetDevice(&prev);
        if (prev != d) CK(cudaSetDevice(d));
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int pick_device()
{
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        fail(HEPFAC_ERR_INTERNAL,
             "no CUDA device available: the B200 build of hepfac matches on the GPU only "
             "(no CPU fallback)");
    }
    int d = 0;
    if (const char* s = std::getenv("HEPFAC_DEVICE")) d = std::atoi(s);
    else cudaGetDevice(&d);
    if (d < 0 || d >= n) invalid("HEPFAC_DEVICE out of range");
    return d;
}

// Dynamic shared memory is a per-kernel-function attribute, and every trie
// with the same kernel choice shares one instantiation: a cap set per trie
// at image time let a small trie lower it below a bigger trie's need (ADVICE
// r1).  Every launch sets the cap to its own trie's size, under one lock
// held across the set and the launch, so concurrent callers with different
// tries cannot lower it between another caller's set and launch, and each
// kernel runs with exactly the shared memory its trie asks for.
std::mutex g_smem_mu;

struct SmemLaunch {
    std::lock_guard<std::mutex> lk{g_smem_mu};
    template <typename F>
    SmemLaunch(F* fn, size_t bytes)
    {
        CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(bytes)));
    }
};

template <typename F>
int occupancy(F* fn, int threads, size_t smem)
{
    SmemLaunch cap(fn, smem);
    int n = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem));
    return n;
}

template <typename T>
T* dev_alloc(size_t count)
{
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    return static_cast<T*>(p);
}

} // namespace

int device_count()
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// ---------------------------------------------------------------------------
// Pinned host memory: match lists and staging buffers are page-locked so the
// D2H of records (and the H2D of staged text) run at PCIe speed and overlap
// the kernels.  cudaHostAlloc costs far more than malloc, so freed blocks are
// kept in a small process-wide pool (HEPFAC_PINNED_POOL_MIB, default 1024 MiB
// of free blocks) and reused by later calls.

namespace {

struct PinnedPool {
    std::mutex mu;
    std::vector<std::pair<size_t, void*>> free; // (capacity, block)
    size_t free_bytes = 0;

    static size_t keep_limit()
    {
        size_t mib = 1024;
        if (const char* s = std::getenv("HEPFAC_PINNED_POOL_MIB")) mib = size_t(std::strtoull(s, nullptr, 10));
        return mib << 20;
    }
    // A block of at least `bytes` (capacities are powers of two >= 1 MiB).
    std::pair<void*, size_t> acquire(size_t bytes)
    {
        size_t cap = size_t(1) << 20;
        while (cap < bytes) cap <<= 1;
        {
            std::lock_guard<std::mutex> lk(mu);
            size_t best = free.size();
            for (size_t i = 0; i < free.size(); ++i)
                if (free[i].first >= cap && (best == free.size() || free[i].first < free[best].first)) best = i;
            if (best != free.size()) {
                auto b = free[best];
                free.erase(free.begin() + long(best));
                free_bytes -= b.first;
                return {b.second, b.first};
            }
        }
        void* p = nullptr;
        const cudaError_t e = cudaHostAlloc(&p, cap, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            cudaGetLastError();
            trim(0); // give the pool's blocks back and retry once
            if (cudaHostAlloc(&p, cap, cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                throw std::bad_alloc();
            }
        }
        return {p, cap};
    }
    void release(void* p, size_t cap)
    {
        if (!p) return;
        {
            std::lock_guard<std::mutex> lk(mu);
            if (free_bytes + cap <= keep_limit()) {
                free.emplace_back(cap, p);
                free_bytes += cap;
                return;
            }
        }
        cudaFreeHost(p);
    }
    void trim(size_t keep)
    {
        std::vector<std::pair<size_t, void*>> drop;
        {
            std::lock_guard<std::mutex> lk(mu);
            while (!free.empty() && free_bytes > keep) {
                drop.push_back(free.back());
                free_bytes -= free.back().first;
                free.pop_back();
            }
        }
        for (auto& b : drop) cudaFreeHost(b.second);
    }
};

PinnedPool& pinned_pool()
{
    static PinnedPool* p = new PinnedPool; // never destroyed: lists may outlive static destructors
    return *p;
}

// Lists up to this many bytes live in ordinary heap memory.
constexpr size_t kPinnedListMin = size_t(1) << 20;

} // namespace

// ---------------------------------------------------------------------------
// MatchList

MatchList::~MatchList() { release(); }

void MatchList::release()
{
    if (pinned) pinned_pool().release(data, cap * sizeof(hepfac_match_t));
    else std::free(data);
    data = nullptr;
    cap = 0;
    pinned = false;
}

void MatchList::allocate(size_t n)
{
    release();
    size = n;
    if (n == 0) return;
    reserve(n);
}

void MatchList::reserve(size_t n)
{
    if (n <= cap) return;
    hepfac_match_t* old = data;
    const bool old_pinned = pinned;
    const size_t old_cap = cap;
    if (n * sizeof(hepfac_match_t) >= kPinnedListMin) {
        auto b = pinned_pool().acquire(n * sizeof(hepfac_match_t));
        data = static_cast<hepfac_match_t*>(b.first);
        cap = b.second / sizeof(hepfac_match_t);
        pinned = true;
    } else {
        data = static_cast<hepfac_match_t*>(std::malloc(n * sizeof(hepfac_match_t)));
        if (!data) {
            data = old;
            throw std::bad_alloc();
        }
        cap = n;
        pinned = false;
    }
    if (old) {
        if (size) std::memcpy(data, old, std::min(size, old_cap) * sizeof(hepfac_match_t));
        if (old_pinned) pinned_pool().release(old, old_cap * sizeof(hepfac_match_t));
        else std::free(old);
    }
}

// ---------------------------------------------------------------------------
// Device image of a trie

using KernelFn = void (*)(gpu::ScanArgs);

struct DeviceTrie {
    int device = 0;
    std::vector<void*> allocs;
    TrieView view{};
    bool grouped = false, identity = false;
    int kw = 0;
    bool pair = false;          // two-pass pipeline: filter pass + candidate-walking pass
    uint32_t filter_mode = 0;   // image.cpp: 1 single, 2 pair, 3 packed symbols, 4 single + L2 bitmap
    void (*filter_fn)(gpu::FilterArgs) = nullptr;
    double filter_pass = 1.0;
    KernelFn kernel = nullptr;
    size_t smem = 0;
    // two-pass pipeline (pair tries, texts >= pipeline_min): filter pass,
    // then the candidate-walking pass; smaller texts use the one-pass `kernel`
    size_t filter_smem = 0;
    int filter_blocks_per_sm = 0;
    KernelFn walk_kernel = nullptr;
    size_t walk_smem = 0;
    int walk_blocks_per_sm = 1;
    uint64_t pipeline_min = 0;
    uint32_t sym_bits = 0; // symbol-key mode: the text is packed before the filter pass
    void (*pack_fn)(const uint8_t*, uint64_t, const uint16_t*, uint32_t*) = nullptr;
    int blocks_per_sm = 1, sm_count = 1;
    // direct-index mode (filter mode 5): pack pass + pfac_dna_kernel
    bool dna = false;
    KernelFn dna_kernel = nullptr;
    size_t dna_smem = 0;
    uint32_t dna_warps = 0;
    uint32_t warps = gpu::kWarps; // per CTA of `kernel`
    uint32_t min_emit = UINT32_MAX, node_count = 0, groups = 0;
    uint64_t reach = 0, filter_paths = 0, device_bytes = 0, private_terminals = 0, keyed_terminals = 0;

    template <typename T>
    const T* upload(const std::vector<T>& v)
    {
        T* d = dev_alloc<T>(v.size());
        allocs.push_back(d);
        if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
        return d;
    }

    ~DeviceTrie()
    {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (void* p : allocs) cudaFree(p);
        if (prev >= 0) cudaSetDevice(prev);
    }
};

namespace {

// HEPFAC_PAIR_PIPELINE=0 keeps pair-filter tries on the fused kernel.
bool pair_pipeline_enabled()
{
    const char* s = std::getenv("HEPFAC_PAIR_PIPELINE");
    return !s || std::strtol(s, nullptr, 10) != 0;
}

// Launches covering fewer starts than this use the one-pass kernel: the
// two-pass pipeline has ~35 us more fixed cost (a second launch, grid
// barriers over more warps), and wins only above ~225 MiB (c3 measurements).
// HEPFAC_PIPELINE_MIN_MIB overrides (0 = always pipeline).
uint64_t pipeline_min_bytes()
{
    uint64_t mib = 256;
    if (const char* s = std::getenv("HEPFAC_PIPELINE_MIN_MIB")) {
        const long v = std::strtol(s, nullptr, 10);
        if (v >= 0) mib = uint64_t(v);
    }
    return mib << 20;
}

KernelFn select_kernel(bool grouped, bool identity, int kw, bool pair)
{
    using namespace gpu;
    // identity byte maps only exist at sigma = 256, i.e. the grouped layout;
    // the pair filter needs k >= 4 (kw 2 or 3)
#define HFB_KW(G, I)                                                                                       \
    {{pfac_scan_kernel<G, I, 0, false>, pfac_scan_kernel<G, I, 0, false>},                                 \
     {pfac_scan_kernel<G, I, 1, false>, pfac_scan_kernel<G, I, 1, false>},                                 \
     {pfac_scan_kernel<G, I, 2, false>, pfac_scan_kernel<G, I, 2, true>},                                  \
     {pfac_scan_kernel<G, I, 3, false>, pfac_scan_kernel<G, I, 3, true>}}
    static const KernelFn table[2][2][4][2] = {{HFB_KW(false, false), HFB_KW(false, false)},
                                               {HFB_KW(true, false), HFB_KW(true, true)}};
#undef HFB_KW
    return table[grouped][identity && grouped][kw][pair ? 1 : 0];
}

// Second pass of the pair pipeline (kw 2 or 3).
KernelFn select_cands_kernel(bool grouped, bool identity, int kw)
{
    using namespace gpu;
#define HFB_C(G, I) {pfac_scan_kernel<G, I, 2, false, true>, pfac_scan_kernel<G, I, 3, false, true>}
    static const KernelFn table[2][2][2] = {{HFB_C(false, false), HFB_C(false, false)},
                                            {HFB_C(true, false), HFB_C(true, true)}};
#undef HFB_C
    return table[grouped][identity && grouped][kw == 3 ? 1 : 0];
}

std::shared_ptr<DeviceTrie> make_device_trie(const Trie& t, int device)
{
    DeviceGuard g(device);
    const GpuImage im = build_gpu_image(t, image_options_from_env());
    auto d = std::make_shared<DeviceTrie>();
    d->device = device;
    d->grouped = im.groups != 0;
    d->identity = im.identity && d->grouped;
    d->kw = im.filter_bits == 0 ? 0 : (im.filter_k == 4 ? 3 : (im.filter_k < 4 ? 1 : 2));
    d->min_emit = im.min_emit;
    d->reach = im.reach;
    d->node_count = im.node_count;
    d->groups = im.groups;
    d->filter_paths = im.filter_paths;
    d->filter_pass = im.filter_pass;
    d->device_bytes = im.device_bytes();
    d->private_terminals = im.private_terminals;
    d->keyed_terminals = im.keyed_terminals;

    TrieView& v = d->view;
    v.nodes = d->upload(im.nodes);
    v.term_id = d->upload(im.term_id);
    v.bucket_of = d->upload(im.bucket_of);
    v.path_id = d->upload(im.path_id);
    v.groups = im.groups;
    v.depth_limit = im.depth_limit;
    v.symtab = d->upload(std::vector<uint16_t>(im.symtab.begin(), im.symtab.end()));
    v.pat_bytes = d->upload(im.pat_bytes);
    v.pat_off = d->upload(im.pat_off);
    v.pat_len = d->upload(im.pat_len);
    v.ht_key = d->upload(im.ht_key);
    v.ht_id = d->upload(im.ht_id);
    v.ht_mask = im.ht_mask;
    v.hmul = im.hmul;
    v.bk_span = d->upload(im.bk_span);
    v.bk_entry = d->upload(im.bk_entry);
    v.filter = d->upload(im.filter);
    v.filter_words = d->kw ? uint32_t(im.filter.size()) : 0u;
    v.filter_bits = im.filter_bits;
    v.filter_k = im.filter_k;
    v.sym_bits = im.sym_bits;
    v.pair_shift = im.pair_shift;
    v.filter2 = d->upload(im.filter2);
    v.key4 = d->upload(im.key4.empty() ? std::vector<uint32_t>(1, 0u) : im.key4);
    v.key4_words = uint32_t(im.key4.size());
    v.filter2_bits = im.filter2_bits;
    v.jump = d->upload(im.jump);
    v.jump_bits = im.jump_bits;
    v.jump_ext = im.jump_ext.empty() ? nullptr : d->upload(im.jump_ext);
    v.min_emit = im.min_emit;
    v.filter_l1 = im.filter_l1.empty() ? nullptr : d->upload(im.filter_l1);
    v.filter_l1_words = uint32_t(im.filter_l1.size());
    if (im.filter_mode == 5) {
        v.dna = d->upload(im.dna);
        v.dna_words = uint32_t(im.dna.size());
        v.dna_keys = im.dna_keys;
        v.dna_pats = im.dna_pats;
        // the pack pass's arithmetic form, when the alphabet follows it
        uint32_t symw = 0;
        bool formula = im.symtab.size() == 256;
        uint32_t count = 0;
        for (uint32_t b = 0; b < 256 && formula; ++b) {
            const uint16_t sy = im.symtab[b];
            if (sy == kNoSym) continue;
            ++count;
            if (sy > 3 || (((b >> 1) ^ (b >> 2)) & 3u) != sy) formula = false;
            else symw |= b << (8 * sy);
        }
        v.dna_symw = formula && count == 4 ? symw : 0u;
        int optin = 0;
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        // 32 warps when the tables and 32 queues fit next to the static
        // shared memory, else 16
        const bool wide = gpu::dna_smem_bytes(im.dna_keys, im.dna_pats, 32) + 1024 <= size_t(optin);
        d->dna_warps = wide ? 32u : 16u;
        d->dna_kernel = wide ? gpu::pfac_dna_kernel<32> : gpu::pfac_dna_kernel<16>;
        d->dna_smem = gpu::dna_smem_bytes(im.dna_keys, im.dna_pats, d->dna_warps);
        d->dna = occupancy(d->dna_kernel, int(d->dna_warps * 32), d->dna_smem) >= 1;
    }

    // one-pass (fused) kernel: always available
    d->kernel = select_kernel(d->grouped, d->identity, d->kw, im.filter_mode == 2);
    d->smem = size_t(v.filter_words) * 4 + gpu::smem_fixed_bytes(false);
    d->blocks_per_sm = occupancy(d->kernel, int(d->warps * 32), d->smem);
    d->blocks_per_sm = std::max(1, d->blocks_per_sm);
    // two-pass pipeline (always for symbol keys: the one-pass kernel reads byte keys)
    d->sym_bits = im.sym_bits;
    d->pair = ((im.filter_mode == 2 || im.filter_mode == 4) && pair_pipeline_enabled()) || im.filter_mode == 3;
    d->filter_mode = im.filter_mode;
    if (d->pair) {
        d->pipeline_min = im.filter_mode == 3 ? 0 : pipeline_min_bytes();
        if (im.filter_mode == 3) {
            d->filter_fn = im.sym_bits == 1 ? gpu::pfac_symbol_filter_kernel<1>
                                            : (im.sym_bits == 2 ? gpu::pfac_symbol_filter_kernel<2>
                                                                : gpu::pfac_symbol_filter_kernel<4>);
            d->pack_fn = im.sym_bits == 1 ? gpu::pfac_pack_symbols_kernel<1>
                                          : (im.sym_bits == 2 ? gpu::pfac_pack_symbols_kernel<2>
                                                              : gpu::pfac_pack_symbols_kernel<4>);
        } else {
            if (im.filter_mode == 4)
                d->filter_fn = d->kw == 3 ? gpu::pfac_l2_filter_kernel<3> : gpu::pfac_l2_filter_kernel<2>;
            else
                d->filter_fn = v.filter2_bits ? gpu::pfac_pair_filter_kernel<true> : gpu::pfac_pair_filter_kernel<false>;
        }
        d->walk_kernel = select_cands_kernel(d->grouped, d->identity, d->kw);
        d->walk_smem = size_t(v.key4_words) * 4 + gpu::smem_fixed_bytes(true); // 4-byte-prefix bitmap, queues
        d->walk_blocks_per_sm = occupancy(d->walk_kernel, int(gpu::kCWarps * 32), d->walk_smem);
        d->walk_blocks_per_sm = std::max(1, d->walk_blocks_per_sm);
        if (im.filter_mode == 4) // the whole shared-memory level, nothing else
            d->filter_smem = size_t(v.filter_l1_words) * 4;
        else // the table, plus the pair form's per-warp step staging
            d->filter_smem = size_t(v.filter_words) * 4 + (im.filter_mode == 3 ? 0 : gpu::pair_smem_fixed_bytes());
        d->filter_blocks_per_sm = occupancy(d->filter_fn, int(gpu::kFThreads), d->filter_smem);
        if (d->filter_blocks_per_sm < 1) fail(HEPFAC_ERR_INTERNAL, "pair filter kernel does not fit an SM");
    }
    CK(cudaDeviceGetAttribute(&d->sm_count, cudaDevAttrMultiProcessorCount, device));
    // A pageable cudaMemcpy may return before its DMA lands, and the scans run
    // on non-blocking streams that do not wait for the legacy stream.
    CK(cudaStreamSynchronize(cudaStreamLegacy));
    return d;
}

} // namespace

Trie::~Trie() = default;

std::shared_ptr<DeviceTrie> Trie::device_image(int device) const
{
    std::lock_guard<std::mutex> lk(dev_mu_);
    if (dev_.size() <= size_t(device)) dev_.resize(size_t(device) + 1);
    if (!dev_[device]) dev_[device] = make_device_trie(*this, device);
    return dev_[device];
}

// ---------------------------------------------------------------------------
// Workspaces: one stream + buffers per concurrent call, pooled per device.

namespace {

struct Workspace {
    int device = 0;
    cudaStream_t stream = nullptr; // kernels (and D2H)
    cudaStream_t copy = nullptr;   // H2D of streamed chunks
    cudaEvent_t ev[6] = {};
    cudaEvent_t h2d_done[2] = {}, kern_done[2] = {};
    uint8_t* d_text = nullptr;
    uint64_t text_cap = 0;
    uint8_t* d_slot[2] = {};       // streamed chunk buffers
    uint64_t slot_cap = 0;
    hepfac_match_t* d_out = nullptr; // final, ordered records
    uint64_t out_cap = 0;
    hepfac_match_t* d_stage = nullptr; // per-warp staging regions
    uint64_t stage_cap = 0, warp_cap = 0;
    uint32_t* d_tile_count = nullptr;
    uint32_t* d_tile_slot = nullptr;
    uint64_t tile_cap = 0, tile_cap2 = 0;
    unsigned long long* d_chunk = nullptr; // one per CTA of the grid
    uint64_t chunk_cap = 0;
    unsigned long long* d_bases = nullptr; // streamed: records before chunk c
    uint64_t bases_cap = 0;
    uint16_t* d_cand = nullptr;            // pair pipeline: per filter warp candidate regions
    uint32_t* d_cand_key = nullptr;        // their first 4 text bytes
    uint64_t cand_alloc = 0, cand_cap = 0, key_alloc = 0;
    uint32_t* d_tile_ccount = nullptr;
    uint32_t* d_tile_cslot = nullptr;
    uint64_t ctile_cap = 0, ctile_cap2 = 0;
    uint32_t* d_tile_region = nullptr;
    uint64_t region_cap = 0;
    uint32_t* d_packed = nullptr; // symbol-key mode: the packed text
    uint64_t packed_cap = 0;
    // [0] max records a warp needed (0 = fits), [1] total of the last launch,
    // [2] error word, [3] zero (base_in of a single launch), [4] its base_out,
    // [5] max candidates a filter warp needed (0 = fits), [6] dynamic unit counter
    unsigned long long* d_small = nullptr;
    unsigned long long* h_small = nullptr; // pinned mirror
    uint4* d_flush = nullptr;
    size_t flush_n16 = 0;
    // streamed hepfac_scan: D2H of each chunk's records on their own stream,
    // a pinned staging ring for pageable callers, per-chunk count mirrors
    cudaStream_t d2h = nullptr;
    static constexpr int kStages = 4;
    uint8_t* h_stage[kStages] = {};
    size_t h_stage_cap = 0;
    cudaEvent_t stage_done[kStages] = {};
    cudaEvent_t cnt_done[2] = {};
    unsigned long long* h_bases = nullptr; // pinned: [0, chunks] running record bases
    size_t h_bases_cap = 0;
    unsigned long long* h_flags = nullptr; // pinned: per slot, d_small[0..5] after its chunk

    explicit Workspace(int dev) : device(dev)
    {
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
        for (auto& e : stage_done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : cnt_done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&h_flags), 2 * 8 * sizeof(unsigned long long), cudaHostAllocDefault));
        for (auto& e : ev) CK(cudaEventCreate(&e));
        for (int k = 0; k < 2; ++k) {
            CK(cudaEventCreateWithFlags(&h2d_done[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&kern_done[k], cudaEventDisableTiming));
        }
        d_small = dev_alloc<unsigned long long>(8);
        CK(cudaMemset(d_small, 0, 8 * sizeof(unsigned long long)));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&h_small), 8 * sizeof(unsigned long long), cudaHostAllocDefault));
    }
    ~Workspace()
    {
        cudaSetDevice(device);
        cudaStreamSynchronize(stream);
        cudaStreamSynchronize(copy);
        cudaStreamSynchronize(d2h);
        for (auto* p : h_stage) pinned_pool().release(p, h_stage_cap);
        if (h_bases) pinned_pool().release(h_bases, h_bases_cap * sizeof(unsigned long long));
        cudaFreeHost(h_flags);
        for (auto& e : stage_done) cudaEventDestroy(e);
        for (auto& e : cnt_done) cudaEventDestroy(e);
        cudaStreamDestroy(d2h);
        for (void* p : {(void*)d_text, (void*)d_slot[0], (void*)d_slot[1], (void*)d_out, (void*)d_stage,
                        (void*)d_tile_count, (void*)d_tile_slot, (void*)d_chunk, (void*)d_bases, (void*)d_small,
                        (void*)d_flush, (void*)d_cand, (void*)d_cand_key, (void*)d_tile_ccount, (void*)d_tile_cslot,
                        (void*)d_tile_region, (void*)d_packed})
            cudaFree(p);
        cudaFreeHost(h_small);
        for (auto& e : ev) cudaEventDestroy(e);
        for (int k = 0; k < 2; ++k) cudaEventDestroy(h2d_done[k]), cudaEventDestroy(kern_done[k]);
        cudaStreamDestroy(copy);
        cudaStreamDestroy(stream);
    }

    template <typename T>
    void regrow(T*& p, uint64_t& cap, uint64_t n)
    {
        if (n <= cap) return;
        CK(cudaStreamSynchronize(stream));
        CK(cudaStreamSynchronize(copy));
        cudaFree(p);
        p = nullptr;
        cap = 0;
        p = dev_alloc<T>(size_t(n));
        cap = n;
    }
    static uint64_t padded(uint64_t bytes) { return ((bytes + 15) & ~uint64_t(15)) + 32; }
    void ensure_text(uint64_t bytes) { regrow(d_text, text_cap, padded(bytes)); }
    void ensure_slots(uint64_t bytes)
    {
        if (padded(bytes) <= slot_cap) return;
        uint64_t c0 = slot_cap, c1 = slot_cap;
        regrow(d_slot[0], c0, padded(bytes));
        regrow(d_slot[1], c1, padded(bytes));
        slot_cap = c0;
    }
    void ensure_out(uint64_t n) { regrow(d_out, out_cap, std::max<uint64_t>(n, 1)); }
    // warp_cap only grows on overflow; the buffer covers warps * warp_cap
    // (never derive warp_cap from the buffer size: grids differ per launch).
    void ensure_stage(uint64_t warps, uint64_t per_warp)
    {
        warp_cap = std::max(warp_cap, per_warp);
        regrow(d_stage, stage_cap, warps * warp_cap);
    }
    void ensure_tiles(uint64_t tiles, uint64_t grid)
    {
        regrow(d_tile_count, tile_cap, tiles);
        regrow(d_tile_slot, tile_cap2, tiles);
        regrow(d_chunk, chunk_cap, grid);
    }
    // cand_cap only grows on overflow, like warp_cap
    void ensure_cand(uint64_t warps, uint64_t per_warp)
    {
        cand_cap = std::max(cand_cap, per_warp);
        regrow(d_cand, cand_alloc, warps * cand_cap);
        regrow(d_cand_key, key_alloc, warps * cand_cap);
    }
    void ensure_ctiles(uint64_t tiles)
    {
        regrow(d_tile_ccount, ctile_cap, tiles);
        regrow(d_tile_cslot, ctile_cap2, tiles);
    }
    // Clears the per-scan accumulators (overflow needs, error word).
    void begin_scan() { CK(cudaMemsetAsync(d_small, 0, 7 * sizeof(unsigned long long), stream)); }

    void ensure_staging(size_t bytes)
    {
        if (bytes <= h_stage_cap) return;
        CK(cudaStreamSynchronize(copy));
        for (auto*& p : h_stage) {
            pinned_pool().release(p, h_stage_cap);
            p = nullptr;
        }
        size_t cap = 0;
        for (auto*& p : h_stage) {
            auto b = pinned_pool().acquire(bytes);
            p = static_cast<uint8_t*>(b.first);
            cap = b.second; // every block of one request has the same capacity
        }
        h_stage_cap = cap;
    }
    void ensure_host_bases(size_t n)
    {
        if (n <= h_bases_cap) return;
        if (h_bases) pinned_pool().release(h_bases, h_bases_cap * sizeof(unsigned long long));
        h_bases = nullptr;
        auto b = pinned_pool().acquire(n * sizeof(unsigned long long));
        h_bases = static_cast<unsigned long long*>(b.first);
        h_bases_cap = b.second / sizeof(unsigned long long);
    }

    // Device bytes held by buffers that regrow on demand.
    uint64_t held_bytes() const
    {
        return text_cap + 2 * slot_cap + out_cap * sizeof(hepfac_match_t) + stage_cap * sizeof(hepfac_match_t) +
               cand_alloc * 2 + key_alloc * 4 + packed_cap * 4;
    }
    // Frees the large regrowable buffers (the next call re-allocates them).
    void shed()
    {
        CK(cudaStreamSynchronize(stream));
        CK(cudaStreamSynchronize(copy));
        CK(cudaStreamSynchronize(d2h));
        auto drop = [](auto*& p, uint64_t& cap) {
            cudaFree(p);
            p = nullptr;
            cap = 0;
        };
        drop(d_text, text_cap);
        drop(d_out, out_cap);
        drop(d_stage, stage_cap);
        warp_cap = 0;
        drop(d_cand, cand_alloc);
        drop(d_cand_key, key_alloc);
        cand_cap = 0;
        drop(d_packed, packed_cap);
        uint64_t c0 = slot_cap, c1 = slot_cap;
        drop(d_slot[0], c0);
        drop(d_slot[1], c1);
        slot_cap = 0;
    }
};

// A pooled workspace keeps at most this many device bytes of regrowable
// buffers when its call returns (HEPFAC_POOL_KEEP_MIB, default 2048); a call
// over a bigger text frees them instead of pinning them for the process.
uint64_t pool_keep_bytes()
{
    uint64_t mib = 2048;
    if (const char* s = std::getenv("HEPFAC_POOL_KEEP_MIB")) mib = std::strtoull(s, nullptr, 10);
    return mib << 20;
}

std::mutex g_pool_mu;
std::vector<std::vector<std::unique_ptr<Workspace>>> g_pool;

struct WorkspaceLease {
    std::unique_ptr<Workspace> ws;
    explicit WorkspaceLease(int dev)
    {
        {
            std::lock_guard<std::mutex> lk(g_pool_mu);
            if (g_pool.size() <= size_t(dev)) g_pool.resize(size_t(dev) + 1);
            if (!g_pool[dev].empty()) {
                ws = std::move(g_pool[dev].back());
                g_pool[dev].pop_back();
            }
        }
        if (!ws) ws = std::make_unique<Workspace>(dev);
    }
    ~WorkspaceLease()
    {
        if (!ws) return;
        int prev = -1;
        cudaGetDevice(&prev);
        if (prev != ws->device) cudaSetDevice(ws->device);
        struct Restore {
            int d;
            ~Restore()
            {
                if (d >= 0) cudaSetDevice(d);
            }
        } restore{prev};
        if (cudaStreamSynchronize(ws->stream) != cudaSuccess || cudaStreamSynchronize(ws->d2h) != cudaSuccess) {
            cudaGetLastError();
            return; // poisoned: drop it
        }
        try {
            if (ws->held_bytes() > pool_keep_bytes()) ws->shed();
        } catch (...) {
            return;
        }
        std::lock_guard<std::mutex> lk(g_pool_mu);
        g_pool[ws->device].push_back(std::move(ws));
    }
    WorkspaceLease(WorkspaceLease&&) = default;
    Workspace* operator->() { return ws.get(); }
    Workspace& operator*() { return *ws; }
};

thread_local ScanStats t_stats;

// Expected records per text byte before the first run tells us better.
uint64_t initial_records(uint64_t bytes) { return std::max<uint64_t>(1u << 14, bytes / 256); }

struct Launch {
    uint64_t n_tiles = 0, grid = 0, warps = 0;
    uint64_t n_ftiles = 0; // pair pipeline: filter tiles (n_tiles counts walk units of kSuper of them)
};

bool pipelined(const DeviceTrie& dt, uint64_t n_own) { return dt.pair && n_own >= dt.pipeline_min; }

Launch plan(const DeviceTrie& dt, uint64_t n_own)
{
    Launch l;
    l.n_tiles = (n_own + gpu::kTile - 1) / gpu::kTile;
    const bool two = pipelined(dt, n_own);
    if (two) {
        l.n_ftiles = l.n_tiles;
        l.n_tiles = (l.n_ftiles + gpu::kSuper - 1) / gpu::kSuper;
    }
    const uint64_t warps = two ? gpu::kCWarps : (dt.dna ? dt.dna_warps : dt.warps);
    const uint64_t bps = two ? dt.walk_blocks_per_sm : (dt.dna ? 1 : dt.blocks_per_sm);
    l.grid = std::min<uint64_t>(uint64_t(dt.sm_count) * bps, std::max<uint64_t>(1, (l.n_tiles + warps - 1) / warps));
    l.warps = l.grid * warps;
    return l;
}

// Enqueue one cooperative launch over device-resident text (no host sync).
// Its records land at [*base_in, *base_in + total) of the output; the launch
// stores *base_in + total to *base_out.
uint32_t enqueue_scan(const DeviceTrie& dt, Workspace& ws, const uint8_t* d_text, uint64_t n_own,
                      uint64_t n_avail, uint64_t g0, const unsigned long long* base_in = nullptr,
                      unsigned long long* base_out = nullptr, cudaEvent_t between = nullptr)
{
    const Launch l = plan(dt, n_own);
    if (!base_in) base_in = ws.d_small + 3, base_out = ws.d_small + 4;
    if (l.n_tiles == 0) {
        CK(cudaMemcpyAsync(base_out, base_in, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, ws.stream));
        return 0;
    }
    ws.ensure_tiles(l.n_tiles, l.grid);
    if (ws.warp_cap == 0) ws.ensure_stage(l.warps, initial_records(n_own) / l.warps + 64);
    ws.ensure_stage(l.warps, ws.warp_cap);
    if (ws.out_cap == 0) ws.ensure_out(initial_records(n_own));
    gpu::ScanArgs a{};
    a.trie = dt.view;
    a.text = d_text;
    a.n_own = n_own;
    a.n_avail = n_avail;
    a.g0 = g0;
    a.out = ws.d_out;
    a.out_cap = ws.out_cap;
    a.stage = ws.d_stage;
    a.warp_cap = ws.warp_cap;
    a.n_tiles = l.n_tiles;
    a.tile_count = ws.d_tile_count;
    a.tile_slot = ws.d_tile_slot;
    a.chunk_sum = ws.d_chunk;
    a.total = ws.d_small + 1;
    a.base_in = base_in;
    a.base_out = base_out;
    a.warp_need = ws.d_small;
    a.err = reinterpret_cast<unsigned int*>(ws.d_small + 2);
    const bool two = pipelined(dt, n_own);
    if (two) {
        const uint64_t fgrid = uint64_t(dt.sm_count) * dt.filter_blocks_per_sm;
        const uint64_t fwarps = fgrid * gpu::kFWarps;
        ws.ensure_ctiles(l.n_ftiles);
        // expected: <= ~1% of starts survive; regions grow on overflow
        if (ws.cand_cap == 0) ws.ensure_cand(fwarps, n_own / 256 / fwarps + 256);
        ws.ensure_cand(fwarps, ws.cand_cap);
        gpu::FilterArgs f{};
        f.table = dt.filter_mode == 4 ? dt.view.filter_l1 : dt.view.filter;
        f.table_words = dt.filter_mode == 4 ? dt.view.filter_l1_words : dt.view.filter_words;
        f.pair_shift = dt.view.pair_shift;
        f.text = d_text;
        f.n_avail = n_avail;
        const uint64_t me = dt.min_emit;
        f.start_end = n_avail >= me ? std::min(n_own, n_avail - me + 1) : 0;
        f.n_tiles = l.n_ftiles;
        f.cand = ws.d_cand;
        f.cand_key = ws.d_cand_key;
        f.cand_cap = ws.cand_cap;
        f.tile_ccount = ws.d_tile_ccount;
        f.tile_cslot = ws.d_tile_cslot;
        f.cand_need = ws.d_small + 5;
        f.filter_k = dt.view.filter_k;
        f.table2 = dt.view.filter2;
        f.table2_bits = dt.view.filter2_bits; // 0 when the image has no L2 level
        if (dt.sym_bits) {
            const uint64_t per = 32 / dt.sym_bits, words = (n_avail + per - 1) / per;
            ws.regrow(ws.d_packed, ws.packed_cap, words + 4);
            CK(cudaMemsetAsync(ws.d_packed + words, 0, 4 * sizeof(uint32_t), ws.stream)); // overhang words
            const unsigned blocks = unsigned(std::min<uint64_t>((words + 255) / 256, uint64_t(dt.sm_count) * 16));
            dt.pack_fn<<<std::max(1u, blocks), 256, 0, ws.stream>>>(d_text, words, dt.view.symtab, ws.d_packed);
            CK(cudaGetLastError());
            f.packed = ws.d_packed;
            a.packed = ws.d_packed;
        }
        {
            SmemLaunch cap(dt.filter_fn, dt.filter_smem);
            dt.filter_fn<<<unsigned(fgrid), gpu::kFThreads, dt.filter_smem, ws.stream>>>(f);
            CK(cudaGetLastError());
        }
        if (between) CK(cudaEventRecord(between, ws.stream));
        // the filter pass already tested the L2 bitmap (single + L2; and the
        // pair filter pass, which tests both bits of its survivors)
        if (dt.filter_mode == 4 || dt.filter_mode == 2) a.trie.filter2_bits = 0;
        a.cand = ws.d_cand;
        a.cand_key = ws.d_cand_key;
        a.cand_cap = ws.cand_cap;
        a.tile_ccount = ws.d_tile_ccount;
        a.tile_cslot = ws.d_tile_cslot;
        a.cand_warps = uint32_t(fwarps);
        a.n_ftiles = l.n_ftiles;
        ws.regrow(ws.d_tile_region, ws.region_cap, l.n_tiles);
        a.tile_region = ws.d_tile_region;
        a.unit_next = ws.d_small + 6;
        // streamed chunks share the counter: zero it before each launch
        CK(cudaMemsetAsync(ws.d_small + 6, 0, sizeof(unsigned long long), ws.stream));
    }
    if (dt.dna) {
        // pack pass (2-bit symbols + validity bits), then the direct-index scan
        const uint64_t vw = (n_avail + 31) / 32 + 4;
        ws.regrow(ws.d_packed, ws.packed_cap, 3 * vw);
        const unsigned blocks = unsigned(std::min<uint64_t>((vw + 255) / 256, uint64_t(dt.sm_count) * 16));
        if (dt.view.dna_symw)
            gpu::pfac_pack_dna_kernel<true><<<std::max(1u, blocks), 256, 0, ws.stream>>>(
                d_text, n_avail, dt.view.symtab, dt.view.dna_symw, ws.d_packed, ws.d_packed + 2 * vw, vw);
        else
            gpu::pfac_pack_dna_kernel<false><<<std::max(1u, blocks), 256, 0, ws.stream>>>(
                d_text, n_avail, dt.view.symtab, 0u, ws.d_packed, ws.d_packed + 2 * vw, vw);
        CK(cudaGetLastError());
        if (between) CK(cudaEventRecord(between, ws.stream));
        a.packed = ws.d_packed;
        a.valid = ws.d_packed + 2 * vw;
        void* dparams[] = {&a};
        SmemLaunch cap(dt.dna_kernel, dt.dna_smem);
        const cudaError_t de = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(dt.dna_kernel),
                                                           dim3(unsigned(l.grid)), dim3(dt.dna_warps * 32), dparams,
                                                           dt.dna_smem, ws.stream);
        if (de != cudaSuccess) {
            cudaGetLastError();
            cuda_fail(de, "pfac_dna_kernel launch");
        }
        return 2;
    }
    void* params[] = {&a};
    SmemLaunch cap(two ? dt.walk_kernel : dt.kernel, two ? dt.walk_smem : dt.smem);
    const cudaError_t e = cudaLaunchCooperativeKernel(
        reinterpret_cast<const void*>(two ? dt.walk_kernel : dt.kernel), dim3(unsigned(l.grid)),
        dim3((two ? gpu::kCWarps : dt.warps) * 32), params, two ? dt.walk_smem : dt.smem, ws.stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        cuda_fail(e, "pfac_scan_kernel launch");
    }
    return two ? 2 : 1;
}

// Reads back the scan's accumulators; true when the results are complete.
// `records` is the word holding the scan's final record count.
bool fetch_small(Workspace& ws, const DeviceTrie& dt, uint64_t n_own, const unsigned long long* records = nullptr)
{
    if (!records) records = ws.d_small + 4;
    CK(cudaMemcpyAsync(ws.h_small, ws.d_small, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ws.stream));
    CK(cudaMemcpyAsync(ws.h_small + 4, records, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ws.stream));
    CK(cudaMemcpyAsync(ws.h_small + 5, ws.d_small + 5, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ws.stream));
    CK(cudaStreamSynchronize(ws.stream));
    if (ws.h_small[2] & 1u) fail(HEPFAC_ERR_INTERNAL, "terminal node spells no dictionary pattern");
    bool ok = true;
    if (ws.h_small[0]) { // some warp's staging region overflowed
        const Launch l = plan(dt, n_own);
        ws.ensure_stage(l.warps, ws.h_small[0] + ws.h_small[0] / 4 + 64);
        ok = false;
    }
    if (ws.h_small[5]) { // some filter warp's candidate region overflowed
        const uint64_t fwarps = uint64_t(dt.sm_count) * std::max(1, dt.filter_blocks_per_sm) * gpu::kFWarps;
        ws.ensure_cand(fwarps, ws.h_small[5] + ws.h_small[5] / 4 + 256);
        ok = false;
    }
    if (ws.h_small[4] > ws.out_cap) {
        ws.ensure_out(ws.h_small[4]);
        ok = false;
    }
    return ok;
}

uint64_t records_of(const Workspace& ws) { return ws.h_small[4]; }

double elapsed_ms(cudaEvent_t a, cudaEvent_t b)
{
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    return double(ms);
}

// Scan of device-resident text, re-run with grown buffers until complete.
uint64_t run_to_completion(const DeviceTrie& dt, Workspace& ws, uint64_t n_own, uint64_t n_avail, uint64_t g0,
                           ScanStats* st)
{
    for (int attempt = 0;; ++attempt) {
        ws.begin_scan();
        if (st) CK(cudaEventRecord(ws.ev[1], ws.stream));
        const uint32_t k = enqueue_scan(dt, ws, ws.d_text, n_own, n_avail, g0);
        if (st) {
            CK(cudaEventRecord(ws.ev[2], ws.stream));
            st->kernel_launches += k;
        }
        if (!k) return 0;
        if (fetch_small(ws, dt, n_own)) return records_of(ws);
        if (st) st->relaunches++;
        if (attempt > 4) fail(HEPFAC_ERR_INTERNAL, "scan buffers keep overflowing");
    }
}

uint64_t stream_chunk_bytes()
{
    uint64_t c = uint64_t(64) << 20;
    if (const char* s = std::getenv("HEPFAC_CHUNK_MIB")) {
        const long v = std::strtol(s, nullptr, 10);
        if (v >= 1 && v <= (1 << 20)) c = uint64_t(v) << 20;
    }
    return c;
}

// Host-to-host copy into a pinned staging buffer on several threads: one
// memcpy thread moves ~10 GB/s, the PCIe Gen5 H2D it feeds ~55 GB/s.
// HEPFAC_COPY_THREADS overrides the count (default: half the host threads, at
// most 8.  On the 16-thread B200 host, with the helpers spinning between
// pieces, 8 beat 12 through hepfac_scan from 1 GiB of pageable text: c2 391-393
// against 360-384 Gbps, c3 421 against 407-419 -- spinning helpers on every
// core starve the driver and the caller).
unsigned copy_threads()
{
    if (const char* s = std::getenv("HEPFAC_COPY_THREADS")) {
        const long v = std::strtol(s, nullptr, 10);
        if (v >= 1) return unsigned(std::min<long>(v, 64));
    }
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    return std::clamp(hw / 2, 1u, 8u);
}

// Persistent helper threads for par_memcpy (spawning threads per 64 MiB
// chunk would cost ~10% of a streamed scan).  Concurrent callers share them.
// A streamed scan hands them one staging piece (2-16 MiB) at a time, so a
// helper that finishes a task spins for a while (HEPFAC_COPY_SPIN_US, default
// 2000: longer than a 16 MiB piece's DMA, which is what the caller waits on
// between pieces once the ring is full) before it sleeps on the condition
// variable, and the caller spins on its batch the same way.  A sleeping
// thread's wake-up per piece cost small pageable scans most (Gbps through
// hepfac_scan, c3 text, sleeping / spinning helpers, scripts/e2e_sizes.py):
// 16 MiB 153 / 182, 64 MiB 217 / 295, 256 MiB 305 / 372, 1 GiB 360-400 / 419
// against 319 / 388 / 430 / 440 from pinned text.
class CopyPool {
public:
    // Runs fn(0..parts-1): the caller runs part 0, helpers the rest (the
    // pool grows to parts - 1 helpers on first need).
    void run(unsigned parts, const std::function<void(unsigned)>& fn)
    {
        struct Batch {
            std::atomic<unsigned> left;
            std::mutex mu;
            std::condition_variable cv;
        } batch;
        batch.left = parts - 1;
        {
            std::lock_guard<std::mutex> lk(mu_);
            while (workers_.size() + 1 < parts) workers_.emplace_back([this] { loop(); });
            for (unsigned i = 1; i < parts; ++i)
                tasks_.push_back([&batch, &fn, i] {
                    fn(i);
                    // decrement under the batch mutex: the caller takes it
                    // before returning, so `batch` (its stack) outlives this
                    std::lock_guard<std::mutex> g(batch.mu);
                    if (batch.left.fetch_sub(1, std::memory_order_acq_rel) == 1) batch.cv.notify_all();
                });
            queued_.fetch_add(parts - 1, std::memory_order_release);
            if (sleepers_) cv_.notify_all();
        }
        fn(0);
        const auto t0 = std::chrono::steady_clock::now();
        while (batch.left.load(std::memory_order_acquire) != 0 && std::chrono::steady_clock::now() - t0 <= spin_)
            relax();
        std::unique_lock<std::mutex> lk(batch.mu); // also waits out the last helper's critical section
        batch.cv.wait(lk, [&] { return batch.left.load(std::memory_order_acquire) == 0; });
    }

private:
    static void relax()
    {
#if defined(__x86_64__) || defined(__i386__)
        __builtin_ia32_pause();
#else
        std::this_thread::yield();
#endif
    }
    static std::chrono::microseconds spin_us()
    {
        long v = 2000;
        if (const char* s = std::getenv("HEPFAC_COPY_SPIN_US")) v = std::clamp(std::strtol(s, nullptr, 10), 0L, 100000L);
        return std::chrono::microseconds(v);
    }
    void loop()
    {
        for (;;) {
            std::function<void()> task;
            const auto t0 = std::chrono::steady_clock::now();
            while (!task) {
                if (queued_.load(std::memory_order_acquire) != 0) {
                    std::lock_guard<std::mutex> lk(mu_);
                    if (!tasks_.empty()) {
                        task = std::move(tasks_.front());
                        tasks_.pop_front();
                        queued_.fetch_sub(1, std::memory_order_relaxed);
                    }
                } else if (std::chrono::steady_clock::now() - t0 > spin_) {
                    std::unique_lock<std::mutex> lk(mu_);
                    ++sleepers_;
                    cv_.wait(lk, [&] { return !tasks_.empty(); });
                    --sleepers_;
                    task = std::move(tasks_.front());
                    tasks_.pop_front();
                    queued_.fetch_sub(1, std::memory_order_relaxed);
                } else {
                    relax();
                }
            }
            task();
        }
    }
    const std::chrono::microseconds spin_ = spin_us();
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> tasks_;
    std::atomic<unsigned> queued_{0};
    unsigned sleepers_ = 0; // guarded by mu_
    std::vector<std::thread> workers_;
};

void par_memcpy(void* dst, const void* src, size_t n)
{
    const size_t kSlice = size_t(256) << 10; // per helper thread at least
    const unsigned T = unsigned(std::min<size_t>(copy_threads(), std::max<size_t>(1, n / kSlice)));
    if (T <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    // helpers detach with the process (never joined: a static destructor
    // must not wait on threads that a late caller may still be using)
    static CopyPool* pool = new CopyPool;
    pool->run(T, [&](unsigned i) {
        const size_t lo = (n * i / T) & ~size_t(4095), hi = i + 1 == T ? n : (n * (i + 1) / T) & ~size_t(4095);
        std::memcpy(static_cast<uint8_t*>(dst) + lo, static_cast<const uint8_t*>(src) + lo, hi - lo);
    });
}

// Staging piece for pageable text: a text's eighth, between 2 and 16 MiB
// (HEPFAC_STAGE_MIB overrides).  Measured on the B200 host (16 threads, 60 MB
// L3; c3 4 GiB / c2 1 GiB / c1 16 MiB, Gbps through hepfac_scan): 2 MiB
// 211 / 210 / 178, 4 MiB 354 / 331 / 77, 8 MiB 414 / 368 / 66, 16 MiB 424 /
// 387 / 61, 64 MiB 374 / 303 / 59 -- against 434 / 431 / 323 from pinned
// text.  Small pieces pay the copy threads' wake-up per piece; whole chunks
// leave the copy and the DMA of a chunk unoverlapped.
uint64_t stage_piece_bytes(uint64_t text_bytes)
{
    if (const char* s = std::getenv("HEPFAC_STAGE_MIB")) {
        const long v = std::strtol(s, nullptr, 10);
        if (v >= 1 && v <= 1024) return uint64_t(v) << 20;
    }
    const uint64_t eighth = ((text_bytes + 7) / 8 + 0xFFFFF) & ~uint64_t(0xFFFFF);
    return std::clamp<uint64_t>(eighth, uint64_t(2) << 20, uint64_t(16) << 20);
}

// Pageable (not page-locked, not device) memory goes through the staging
// ring; pinned host memory and device pointers are copied from directly.
bool is_pageable(const void* p)
{
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// Streamed scan of host text.  Chunks of starts (with the `halo` of right
// context their walks may read) go H2D on the copy stream into two device
// slots while the previous chunk's launch runs on the compute stream; each
// launch places its records right after the previous chunk's (device-side
// running base), so the output is ordered without host syncs between chunks.
// Pageable text is copied (several host threads) piece by piece into a ring
// of kStages small pinned buffers, each piece's DMA queued as soon as it is
// copied, so the host copy of piece p+1 overlaps the DMA of piece p.  With a
// `sink`, chunk c's records
// go D2H (own stream) into the sink as soon as its kernel has finished,
// overlapping chunks c+1...; without one they stay in ws.d_out.
uint64_t stream_scan(const DeviceTrie& dt, Workspace& ws, const uint8_t* text, uint64_t avail, uint64_t owned,
                     uint64_t g0, uint64_t halo, MatchList* sink, ScanStats& st)
{
    const bool stage = is_pageable(text);
    const uint64_t C = stream_chunk_bytes();
    const uint64_t n = (owned + C - 1) / C;
    const uint64_t slot_bytes = std::min(avail, C + halo);
    const uint64_t piece = stage_piece_bytes(avail);
    ws.ensure_slots(slot_bytes);
    if (stage) ws.ensure_staging(piece);
    ws.regrow(ws.d_bases, ws.bases_cap, n + 1);
    ws.ensure_host_bases(n + 1);
    if (ws.out_cap < initial_records(owned)) ws.ensure_out(initial_records(owned));
    st.staged = stage;
    for (int attempt = 0;; ++attempt) {
        ws.begin_scan();
        CK(cudaMemsetAsync(ws.d_bases, 0, sizeof(unsigned long long), ws.stream));
        ws.h_bases[0] = 0;
        if (sink) sink->size = 0;
        CK(cudaEventRecord(ws.ev[0], ws.stream));
        CK(cudaStreamWaitEvent(ws.copy, ws.ev[0], 0));
        bool overflow = false;
        uint64_t pieces = 0; // staged pieces queued so far (ring position)
        // chunk k's base and overflow words are on the host once cnt_done fires
        auto drain = [&](uint64_t k) {
            const int slot = int(k & 1);
            CK(cudaEventSynchronize(ws.cnt_done[slot]));
            const unsigned long long* f = ws.h_flags + 8 * slot;
            if (f[2] & 1u) fail(HEPFAC_ERR_INTERNAL, "terminal node spells no dictionary pattern");
            const uint64_t b0 = ws.h_bases[k], b1 = ws.h_bases[k + 1];
            if (overflow || f[0] || f[5] || b1 > ws.out_cap) {
                overflow = true; // finish the pass, grow, re-run (fetch_small)
                return;
            }
            if (!sink || b1 == b0) return;
            if (b1 > sink->cap) { // extrapolate from the chunks so far
                CK(cudaStreamSynchronize(ws.d2h));
                sink->size = b0;
                const double per = double(b1) / double(k + 1);
                sink->reserve(std::max<uint64_t>(b1, uint64_t(per * double(n) * 1.125) + 1024));
            }
            CK(cudaMemcpyAsync(sink->data + b0, ws.d_out + b0, size_t(b1 - b0) * sizeof(hepfac_match_t),
                               cudaMemcpyDeviceToHost, ws.d2h));
            sink->size = b1;
        };
        for (uint64_t c = 0; c < n; ++c) {
            const int slot = int(c & 1);
            const uint64_t lo = c * C, own = std::min(C, owned - lo), bytes = std::min(avail - lo, own + halo);
            const uint8_t* src = text + lo;
            if (c >= 2) CK(cudaStreamWaitEvent(ws.copy, ws.kern_done[slot], 0));
            if (stage) {
                for (uint64_t off = 0; off < bytes; off += piece, ++pieces) {
                    const uint64_t len = std::min(piece, bytes - off);
                    const int r = int(pieces % Workspace::kStages);
                    if (pieces >= uint64_t(Workspace::kStages)) CK(cudaEventSynchronize(ws.stage_done[r]));
                    par_memcpy(ws.h_stage[r], src + off, size_t(len));
                    CK(cudaMemcpyAsync(ws.d_slot[slot] + off, ws.h_stage[r], size_t(len), cudaMemcpyHostToDevice,
                                       ws.copy));
                    CK(cudaEventRecord(ws.stage_done[r], ws.copy));
                }
            } else {
                CK(cudaMemcpyAsync(ws.d_slot[slot], src, size_t(bytes), cudaMemcpyDefault, ws.copy));
            }
            CK(cudaEventRecord(ws.h2d_done[slot], ws.copy));
            CK(cudaStreamWaitEvent(ws.stream, ws.h2d_done[slot], 0));
            if (c == 0) CK(cudaEventRecord(ws.ev[1], ws.stream));
            st.kernel_launches +=
                enqueue_scan(dt, ws, ws.d_slot[slot], own, bytes, g0 + lo, ws.d_bases + c, ws.d_bases + c + 1);
            CK(cudaEventRecord(ws.kern_done[slot], ws.stream));
            CK(cudaMemcpyAsync(ws.h_bases + c + 1, ws.d_bases + c + 1, sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, ws.stream));
            CK(cudaMemcpyAsync(ws.h_flags + 8 * slot, ws.d_small, 6 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, ws.stream));
            CK(cudaEventRecord(ws.cnt_done[slot], ws.stream));
            if (c >= 1) drain(c - 1);
        }
        CK(cudaEventRecord(ws.ev[2], ws.stream));
        drain(n - 1);
        st.chunks = uint32_t(n);
        if (!overflow) return ws.h_bases[n];
        CK(cudaStreamSynchronize(ws.d2h));
        if (fetch_small(ws, dt, C, ws.d_bases + n)) // cannot happen: some word said overflow
            fail(HEPFAC_ERR_INTERNAL, "streamed scan overflow not confirmed by the device");
        st.relaunches++;
        if (attempt > 4) fail(HEPFAC_ERR_INTERNAL, "scan buffers keep overflowing");
    }
}

// One shard of starts on one device.  With a `sink` the records land in it
// (overlapped D2H) and the workspace returns to the pool; without, `keep`
// holds the workspace and its device-resident records for a later copy.
struct ShardJob {
    std::unique_ptr<WorkspaceLease> ws;
    uint64_t total = 0;
    ScanStats st;
};

void run_shard(const Trie& t, const uint8_t* text, uint64_t avail, uint64_t owned, uint64_t g0, int device,
               MatchList* sink, ShardJob& job)
{
    ScanStats& st = job.st;
    st = ScanStats{};
    st.bytes = owned;
    if (owned == 0) return;
    const int dev = device >= 0 ? device : pick_device();
    st.device = dev;
    DeviceGuard g(dev);
    auto dt = t.device_image(dev);
    if (dt->min_emit == UINT32_MAX || avail < dt->min_emit) return;
    job.ws = std::make_unique<WorkspaceLease>(dev);
    Workspace& ws = **job.ws;
    uint64_t total;
    if (dt->reach != UINT64_MAX) {
        total = stream_scan(*dt, ws, text, avail, owned, g0, dt->reach ? dt->reach - 1 : 0, sink, st);
    } else { // cyclic loaded trie: walks have no bounded halo, so the text goes in one piece
        ws.ensure_text(avail);
        CK(cudaEventRecord(ws.ev[0], ws.stream));
        CK(cudaMemcpyAsync(ws.d_text, text, size_t(avail), cudaMemcpyDefault, ws.stream));
        total = run_to_completion(*dt, ws, owned, avail, g0, &st);
        st.chunks = 1;
        if (sink) {
            sink->allocate(size_t(total));
            if (total)
                CK(cudaMemcpyAsync(sink->data, ws.d_out, size_t(total) * sizeof(hepfac_match_t),
                                   cudaMemcpyDeviceToHost, ws.d2h));
        }
    }
    job.total = total;
    CK(cudaEventRecord(ws.ev[3], ws.d2h));
    CK(cudaStreamSynchronize(ws.d2h));
    CK(cudaStreamSynchronize(ws.stream));
    st.h2d_ms = elapsed_ms(ws.ev[0], ws.ev[1]);  // streamed: first chunk only
    st.kernel_ms = elapsed_ms(ws.ev[1], ws.ev[2]); // streamed: kernels overlapped with later copies
    st.d2h_ms = std::max(0.0, elapsed_ms(ws.ev[2], ws.ev[3]));
    st.total_ms = elapsed_ms(ws.ev[0], ws.ev[3]);
    st.matches = total;
    if (sink) job.ws.reset(); // back to the pool
}

std::unique_ptr<MatchList> scan_one(const Trie& t, const uint8_t* text, uint64_t avail, uint64_t owned, uint64_t g0,
                                    int device = -1)
{
    auto out = std::make_unique<MatchList>();
    ShardJob job;
    run_shard(t, text, avail, owned, g0, device, out.get(), job);
    out->size = size_t(job.total);
    t_stats = job.st;
    return out;
}

} // namespace

const ScanStats& last_scan_stats() { return t_stats; }

// HEPFAC_DEVICES: devices one hepfac_scan call shards its text over
// ("all", or a comma list such as "0,1,2,3"; a device may repeat).  Unset:
// the single device of pick_device().
std::vector<int> scan_devices()
{
    const char* s = std::getenv("HEPFAC_DEVICES");
    if (!s || !*s) return {pick_device()};
    const int n = device_count();
    if (n <= 0) pick_device(); // fails with the no-device message
    std::vector<int> devs;
    if (std::string(s) == "all") {
        for (int d = 0; d < n; ++d) devs.push_back(d);
        return devs;
    }
    for (const char* p = s; *p;) {
        char* end = nullptr;
        const long d = std::strtol(p, &end, 10);
        if (end == p || d < 0 || d >= n) invalid("HEPFAC_DEVICES lists an invalid device");
        devs.push_back(int(d));
        p = *end == ',' ? end + 1 : end;
        if (*end && *end != ',') invalid("HEPFAC_DEVICES must be 'all' or a comma-separated device list");
    }
    if (devs.empty()) invalid("HEPFAC_DEVICES lists no device");
    return devs;
}

// Multi-GPU hepfac_scan: contiguous shards of starts, each with
// the halo its walks may read, scanned concurrently (one host thread per
// shard) with their records left on their devices.  The exclusive scan of
// the per-shard counts gives each shard's offset in the one host list, and
// every device copies its sorted records straight to out + prefix[g]: shard
// order is the whole list's order.
std::unique_ptr<MatchList> gpu_scan(const Trie& t, const uint8_t* text, uint64_t bytes)
{
    if (bytes == 0) return scan_one(t, text, 0, 0, 0); // empty: never touches a device
    const std::vector<int> devs = scan_devices();
    constexpr uint64_t kMinShard = uint64_t(16) << 20;
    const uint64_t G = std::min<uint64_t>(devs.size(), std::max<uint64_t>(1, bytes / kMinShard));
    if (G <= 1) return scan_one(t, text, bytes, bytes, 0, devs[0]);
    const uint64_t reach = t.device_image(devs[0])->reach;
    if (reach == UINT64_MAX) return scan_one(t, text, bytes, bytes, 0, devs[0]); // cyclic: no halo bound
    const uint64_t halo = reach ? reach - 1 : 0;
    // (declared before the jobs: on an error the jobs' workspaces synchronize
    // their streams before the list their copies target is freed)
    auto out = std::make_unique<MatchList>();
    std::vector<ShardJob> jobs(G);
    std::vector<std::exception_ptr> errs(G);
    auto parallel = [&](auto&& fn) {
        std::vector<std::thread> pool;
        for (uint64_t g = 0; g < G; ++g)
            pool.emplace_back([&, g] {
                try {
                    fn(g);
                } catch (...) {
                    errs[g] = std::current_exception();
                }
            });
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    };
    parallel([&](uint64_t g) {
        const uint64_t lo = bytes * g / G, hi = bytes * (g + 1) / G;
        const uint64_t avail = std::min(bytes - lo, hi - lo + halo);
        run_shard(t, text + lo, avail, hi - lo, lo, devs[g], nullptr, jobs[g]);
    });
    std::vector<uint64_t> prefix(G + 1, 0); // the count exchange: exclusive scan of shard totals
    for (uint64_t g = 0; g < G; ++g) prefix[g + 1] = prefix[g] + jobs[g].total;
    out->allocate(size_t(prefix[G]));
    parallel([&](uint64_t g) {
        if (!jobs[g].total) return;
        Workspace& ws = **jobs[g].ws;
        DeviceGuard dg(ws.device);
        CK(cudaMemcpyAsync(out->data + prefix[g], ws.d_out, size_t(jobs[g].total) * sizeof(hepfac_match_t),
                           cudaMemcpyDeviceToHost, ws.d2h));
        CK(cudaStreamSynchronize(ws.d2h));
    });
    ScanStats st;
    st.bytes = bytes;
    st.device = devs[0];
    for (uint64_t g = 0; g < G; ++g) {
        const ScanStats& s = jobs[g].st;
        st.kernel_launches += s.kernel_launches;
        st.chunks += s.chunks;
        st.relaunches += s.relaunches;
        st.staged = st.staged || s.staged;
        st.h2d_ms = std::max(st.h2d_ms, s.h2d_ms);
        st.kernel_ms = std::max(st.kernel_ms, s.kernel_ms);
        st.d2h_ms = std::max(st.d2h_ms, s.d2h_ms);
        st.total_ms = std::max(st.total_ms, s.total_ms);
    }
    st.matches = prefix[G];
    t_stats = st;
    return out;
}

std::unique_ptr<MatchList> gpu_scan_shard(const Trie& t, const uint8_t* text, uint64_t avail, uint64_t owned,
                                          uint64_t g0)
{
    if (owned > avail) invalid("shard owns more starts than it has bytes");
    return scan_one(t, text, avail, owned, g0);
}

void trim_pools()
{
    std::vector<std::unique_ptr<Workspace>> drop;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (auto& v : g_pool)
            for (auto& w : v) drop.push_back(std::move(w));
        g_pool.clear();
    }
    drop.clear(); // workspace destructors free device buffers and return pinned blocks
    pinned_pool().trim(0);
}

// The halo is a property of the trie (its longest walk), computed by the
// host-side image builder, so shard planning works on hosts without a GPU
// (e.g. a coordinator, or the CPU tests of the multi-process path).
uint64_t gpu_halo(const Trie& t)
{
    uint64_t reach;
    if (device_count() > 0) reach = t.device_image(pick_device())->reach;
    else reach = build_gpu_image(t, image_options_from_env()).reach;
    return reach == UINT64_MAX ? UINT64_MAX : (reach ? reach - 1 : 0);
}

LayoutInfo layout_info(const Trie& t)
{
    const int dev = pick_device();
    auto d = t.device_image(dev);
    LayoutInfo li{};
    li.node_count = d->node_count;
    li.groups = d->groups;
    li.record_bytes = d->groups ? 16 * d->groups : 8;
    li.filter_k = d->view.filter_k;
    li.filter_bits = d->view.filter_bits;
    li.min_emit = d->min_emit;
    li.smem_bytes = uint32_t(d->smem);
    li.blocks_per_sm = uint32_t(d->blocks_per_sm);
    li.sm_count = uint32_t(d->sm_count);
    li.identity = d->identity;
    li.filter_paths = d->filter_paths;
    li.reach = d->reach;
    li.device_bytes = d->device_bytes;
    li.private_terminals = d->private_terminals;
    li.keyed_terminals = d->keyed_terminals;
    li.filter_mode = d->dna ? 5u : (d->kw == 0 ? 0u : (d->filter_mode == 5 ? 1u : d->filter_mode));
    li.filter_pass_ppm = uint32_t(std::min(1.0, d->filter_pass) * 1e6);
    li.filter2_bits = d->view.filter2_bits;
    return li;
}

// ---------------------------------------------------------------------------
// run_throughput (reference bench.cpp:52-78)

Throughput gpu_run_throughput(const Trie& t, const uint8_t* text, uint64_t bytes, uint32_t runs)
{
    if (runs < 1) invalid("runs must be >= 1");
    if (bytes == 0) invalid("empty corpus");
    Throughput r;
    const int dev = pick_device();
    DeviceGuard g(dev);
    auto dt = t.device_image(dev);
    WorkspaceLease ws(dev);
    ws->ensure_text(bytes);
    CK(cudaMemcpyAsync(ws->d_text, text, size_t(bytes), cudaMemcpyHostToDevice, ws->stream));
    CK(cudaStreamSynchronize(ws->stream));
    // A trie that cannot match here launches nothing, but its runs are still
    // timed (event pairs on the stream), so the report never carries seconds
    // of 0 (the reference always times its runs, bench.cpp:64-76).
    const bool can_match = dt->min_emit != UINT32_MAX && bytes >= dt->min_emit;
    if (can_match) run_to_completion(*dt, *ws, bytes, bytes, 0, nullptr); // warm-up, untimed; sizes the buffers
    std::vector<hepfac_match_t> host;
    double sum_scan = 0, sum_merge = 0;
    for (uint32_t i = 0; i < runs; ++i) {
        ws->begin_scan();
        CK(cudaEventRecord(ws->ev[0], ws->stream));
        if (can_match) enqueue_scan(*dt, *ws, ws->d_text, bytes, bytes, 0);
        CK(cudaEventRecord(ws->ev[1], ws->stream));
        if (can_match && !fetch_small(*ws, *dt, bytes))
            fail(HEPFAC_ERR_INTERNAL, "scan buffers overflowed after warm-up");
        r.matches = can_match ? records_of(*ws) : 0;
        host.resize(size_t(r.matches));
        CK(cudaEventRecord(ws->ev[2], ws->stream));
        if (r.matches)
            CK(cudaMemcpyAsync(host.data(), ws->d_out, size_t(r.matches) * sizeof(hepfac_match_t),
                               cudaMemcpyDeviceToHost, ws->stream));
        CK(cudaEventRecord(ws->ev[3], ws->stream));
        CK(cudaStreamSynchronize(ws->stream));
        sum_scan += elapsed_ms(ws->ev[0], ws->ev[1]) / 1e3;
        sum_merge += elapsed_ms(ws->ev[2], ws->ev[3]) / 1e3;
    }
    r.seconds = sum_scan / runs;
    r.merge_seconds = sum_merge / runs;
    return r;
}

// ---------------------------------------------------------------------------
// Device-resident benchmark session

struct Session {
    std::shared_ptr<DeviceTrie> dt;
    std::unique_ptr<Workspace> ws;
    uint64_t bytes = 0, matches = 0, offset = 0, owned = 0;
    bool complete = false, split = false, sized = false;
    uint32_t last_iterations = 0;
    std::vector<cudaEvent_t> evs;
    ~Session()
    {
        if (!ws) return;
        cudaSetDevice(ws->device);
        for (auto e : evs) cudaEventDestroy(e);
    }
};

Session* session_create(const Trie& t, const uint8_t* text, uint64_t bytes, uint64_t offset, uint64_t owned)
{
    if (bytes == 0) invalid("empty corpus");
    if (owned > bytes) invalid("shard owns more starts than it has bytes");
    const int dev = pick_device();
    DeviceGuard g(dev);
    auto s = std::make_unique<Session>();
    s->dt = t.device_image(dev);
    s->ws = std::make_unique<Workspace>(dev);
    s->bytes = bytes;
    s->offset = offset;
    s->owned = owned;
    s->ws->ensure_text(bytes);
    CK(cudaMemcpyAsync(s->ws->d_text, text, size_t(bytes), cudaMemcpyHostToDevice, s->ws->stream));
    CK(cudaStreamSynchronize(s->ws->stream));
    return s.release();
}

void session_run(Session* s, uint32_t iterations, int flush_l2, double* ms_each)
{
    Workspace& ws = *s->ws;
    DeviceGuard g(ws.device);
    const DeviceTrie& dt = *s->dt;
    const bool can_match = dt.min_emit != UINT32_MAX && s->bytes >= dt.min_emit;
    if (flush_l2 && !ws.d_flush) {
        int l2 = 0;
        CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ws.device));
        ws.flush_n16 = size_t(l2) * 2 / 16;
        ws.d_flush = dev_alloc<uint4>(ws.flush_n16);
    }
    while (s->evs.size() < 3 * size_t(iterations)) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        s->evs.push_back(e);
    }
    // The first run sizes every buffer (candidates, staging, output) with
    // untimed scans until one completes, so timed iterations never overflow.
    if (can_match && !s->sized) run_to_completion(dt, ws, s->owned, s->bytes, s->offset, nullptr);
    s->sized = true;
    ws.begin_scan();
    for (uint32_t i = 0; i < iterations; ++i) {
        if (flush_l2)
            gpu::l2_flush_kernel<<<dt.sm_count * 4, 512, 0, ws.stream>>>(ws.d_flush, ws.flush_n16, i);
        CK(cudaEventRecord(s->evs[3 * i], ws.stream));
        if (can_match) enqueue_scan(dt, ws, ws.d_text, s->owned, s->bytes, s->offset, nullptr, nullptr, s->evs[3 * i + 1]);
        CK(cudaEventRecord(s->evs[3 * i + 2], ws.stream));
    }
    s->last_iterations = iterations;
    s->split = can_match && (pipelined(dt, s->owned) || dt.dna);
    s->complete = !can_match || fetch_small(ws, dt, s->owned); // grows buffers for the next run
    s->matches = can_match ? records_of(ws) : 0;
    for (uint32_t i = 0; i < iterations; ++i)
        if (ms_each) ms_each[i] = elapsed_ms(s->evs[3 * i], s->evs[3 * i + 2]);
}

void session_split(Session* s, uint32_t n, double* first_ms, double* second_ms, uint32_t* kernels_per_scan)
{
    DeviceGuard g(s->ws->device);
    if (kernels_per_scan)
        *kernels_per_scan = s->dt->dna ? 2u : (pipelined(*s->dt, s->owned) ? (s->dt->sym_bits ? 3u : 2u) : 1u);
    n = std::min(n, s->last_iterations);
    for (uint32_t i = 0; i < n; ++i) {
        const double total = elapsed_ms(s->evs[3 * i], s->evs[3 * i + 2]);
        const double first = s->split ? elapsed_ms(s->evs[3 * i], s->evs[3 * i + 1]) : total;
        if (first_ms) first_ms[i] = first;
        if (second_ms) second_ms[i] = total - first;
    }
}

uint64_t session_matches(Session* s) { return s->matches; }

std::unique_ptr<MatchList> session_fetch(Session* s)
{
    Workspace& ws = *s->ws;
    DeviceGuard g(ws.device);
    if (!s->complete) fail(HEPFAC_ERR_STATE, "session results overflowed: run again before fetching");
    auto out = std::make_unique<MatchList>();
    out->allocate(size_t(s->matches));
    if (s->matches)
        CK(cudaMemcpy(out->data, ws.d_out, size_t(s->matches) * sizeof(hepfac_match_t), cudaMemcpyDeviceToHost));
    return out;
}

void session_destroy(Session* s) { delete s; }

} // namespace hfb

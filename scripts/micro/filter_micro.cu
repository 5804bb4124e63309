// filter_micro.cu -- stand-alone ceiling test of the pair start filter
// (level 1 + in-lane level 2) over device-resident random text, without the
// walk/queue machinery.  Not part of the library; used to choose the kernel
// shape (warps per SM, direct loads vs TMA staging).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o filter_micro filter_micro.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr uint32_t kPairMul = 0x2545F491u << 8;
__host__ __device__ inline uint32_t pair_word(uint32_t m, uint32_t wb) { return (m * kPairMul) >> (32 - wb); }

__device__ __forceinline__ uint32_t lds(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    filt(const uint4* __restrict__ text, uint64_t n16, const uint32_t* __restrict__ table, uint32_t wb,
         unsigned long long* out, int level2)
{
    extern __shared__ uint32_t s_tab[];
    for (uint32_t i = threadIdx.x; i < (1u << wb); i += blockDim.x) s_tab[i] = table[i];
    __syncthreads();
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
    const uint32_t lane = threadIdx.x & 31, gw = blockIdx.x * WARPS + (threadIdx.x >> 5), W = gridDim.x * WARPS;
    const uint32_t shift = 32 - wb;
    uint32_t count = 0;
    // each warp: 512-byte chunks, lane owns 16 bytes; overhang word from lane+1
    const uint64_t chunks = n16 / 32;
    uint4 cur = chunks > gw ? __ldg(text + uint64_t(gw) * 32 + lane) : make_uint4(0, 0, 0, 0);
    for (uint64_t c = gw; c < chunks; c += W) {
        const uint64_t cn = c + W;
        uint4 nxt = cn < chunks ? __ldg(text + cn * 32 + lane) : make_uint4(0, 0, 0, 0);
        uint32_t ov = __shfl_sync(0xFFFFFFFFu, cur.x, (lane + 1) & 31);
        const uint32_t w[5] = {cur.x, cur.y, cur.z, cur.w, ov};
        uint32_t m0 = 0, m1 = 0;
#pragma unroll
        for (int i = 1; i < 16; i += 2) {
            auto win = [&](int n) -> uint32_t {
                return (n & 3) ? __funnelshift_r(w[n >> 2], w[(n >> 2) + 1], 8 * (n & 3)) : w[n >> 2];
            };
            const uint32_t mid = win(i), a = win(i - 1), b = win(i + 3);
            const uint32_t word = lds(base + (((mid * kPairMul) >> shift) << 2));
            uint32_t& m = i < 8 ? m0 : m1;
            m = __funnelshift_l(__funnelshift_l(0u, word, a), m, 1);
            m = __funnelshift_l(__funnelshift_l(0u, word, b), m, 1);
        }
        uint32_t mask = (m0 << 8) | m1; // start j at bit 15 - j
        if (level2 == 2) {
            // stage this lane's 16 + 4 bytes, compact candidates, test 32 per round
            uint8_t* stg = reinterpret_cast<uint8_t*>(s_tab + (1u << wb)) + (threadIdx.x >> 5) * (512 + 16 + 1024);
            uint16_t* q = reinterpret_cast<uint16_t*>(stg + 512 + 16);
            *reinterpret_cast<uint4*>(stg + 16 * lane) = cur;
            if (lane == 31) *reinterpret_cast<uint32_t*>(stg + 512) = ov;
            const uint32_t cnt = __popc(mask);
            uint32_t incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= uint32_t(d)) incl += u;
            }
            const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
            uint32_t at = incl - cnt;
            for (uint32_t cm = mask; cm; cm &= cm - 1) q[at++] = uint16_t(16 * lane + 15 - (__ffs(cm) - 1));
            __syncwarp();
            uint32_t keep_n = 0;
            for (uint32_t r0 = 0; r0 < tot; r0 += 32) {
                bool keep = false;
                if (r0 + lane < tot) {
                    const uint32_t off = q[r0 + lane];
                    const uint32_t* wp = reinterpret_cast<const uint32_t*>(stg + (off & ~3u));
                    const uint32_t y = __funnelshift_r(wp[0], wp[1], 8 * off);
                    const bool odd = off & 1;
                    const uint32_t mid = odd ? y >> 8 : y, amt = odd ? y : y >> 24;
                    const uint32_t word = lds(base + (((mid * kPairMul) >> shift) << 2));
                    keep = int32_t(word << (amt & 31)) < 0;
                }
                keep_n += __popc(__ballot_sync(0xFFFFFFFFu, keep));
            }
            __syncwarp();
            count += lane == 0 ? keep_n : 0;
            mask = 0;
        } else if (level2) {
            uint32_t keep = 0;
            for (uint32_t cm = mask; cm; cm &= cm - 1) {
                const uint32_t bit = __ffs(cm) - 1, j = 15 - bit;
                const uint32_t q = j >> 2;
                uint32_t lo = w[0], hi = w[1];
#pragma unroll
                for (int k = 1; k < 4; ++k)
                    if (q == uint32_t(k)) lo = w[k], hi = w[k + 1];
                const uint32_t y = __funnelshift_r(lo, hi, 8 * j);
                const bool odd = j & 1;
                const uint32_t mid = odd ? y >> 8 : y, amt = odd ? y : y >> 24;
                const uint32_t word = lds(base + (((mid * kPairMul) >> shift) << 2));
                if (int32_t(word << (amt & 31)) < 0) keep |= 1u << bit;
            }
            mask = keep;
        }
        count += __popc(mask);
        cur = nxt;
    }
    for (int d = 16; d; d >>= 1) count += __shfl_xor_sync(0xFFFFFFFFu, count, d);
    if (lane == 0) atomicAdd(out, count);
}

__global__ void fill(uint4* t, uint64_t n16, uint32_t seed)
{
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n16; i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        uint32_t v[4];
        for (int k = 0; k < 4; ++k) {
            x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
            v[k] = uint32_t(x);
        }
        t[i] = make_uint4(v[0], v[1], v[2], v[3]);
    }
}

template <int WARPS>
void run(const uint4* d_text, uint64_t n16, const uint32_t* d_tab, uint32_t wb, int level2)
{
    unsigned long long* d_out;
    cudaMalloc(&d_out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = (size_t(4) << wb) + (level2 == 2 ? WARPS * (512 + 16 + 1024) : 0);
    cudaFuncSetAttribute(filt<WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    float best = 1e9;
    unsigned long long cnt = 0;
    for (int it = 0; it < 8; ++it) {
        cudaMemset(d_out, 0, 8);
        cudaEventRecord(e0);
        filt<WARPS><<<sms, WARPS * 32, smem>>>(d_text, n16, d_tab, wb, d_out, level2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 2 && ms < best) best = ms;
        cudaMemcpy(&cnt, d_out, 8, cudaMemcpyDeviceToHost);
    }
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, filt<WARPS>);
    printf("warps=%d level2=%d regs=%d: %.3f ms  %.1f GB/s  survivors=%llu (%.4f%%)  err=%s\n", WARPS, level2,
           fa.numRegs, best, n16 * 16 / best / 1e6, cnt, 100.0 * cnt / (n16 * 16.0),
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d_out);
}


// Batched second level: 4 consecutive 512-byte chunks per warp keep their
// first-level masks in registers and their text in a per-warp smem staging
// area; one packed scan, one compaction, full 32-lane test rounds.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    filt_batch(const uint4* __restrict__ text, uint64_t n16, const uint32_t* __restrict__ table, uint32_t wb,
               unsigned long long* out)
{
    extern __shared__ uint32_t s_tab[];
    for (uint32_t i = threadIdx.x; i < (1u << wb); i += blockDim.x) s_tab[i] = table[i];
    __syncthreads();
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * WARPS + warp, W = gridDim.x * WARPS;
    const uint32_t shift = 32 - wb;
    constexpr int B = 4;
    uint8_t* stg = reinterpret_cast<uint8_t*>(s_tab + (1u << wb)) + warp * (B * 528 + 2048 * B / 4);
    uint16_t* q = reinterpret_cast<uint16_t*>(stg + B * 528);
    uint32_t count = 0;
    const uint64_t chunks = n16 / 32; // 512-byte chunks; a warp takes B consecutive ones per step
    const uint64_t steps = chunks / B;
    for (uint64_t st = gw; st < steps; st += W) {
        uint4 cur[B];
#pragma unroll
        for (int b = 0; b < B; ++b) cur[b] = __ldg(text + (st * B + b) * 32 + lane);
        uint32_t packed = 0;
        uint32_t masks[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            uint32_t ov = __shfl_sync(0xFFFFFFFFu, cur[b].x, (lane + 1) & 31);
            const uint32_t nx = __shfl_sync(0xFFFFFFFFu, cur[b < B - 1 ? b + 1 : b].x, 0);
            if (lane == 31) ov = b + 1 < B ? nx : 0u;
            const uint32_t w[5] = {cur[b].x, cur[b].y, cur[b].z, cur[b].w, ov};
            *reinterpret_cast<uint4*>(stg + b * 528 + 16 * lane) = cur[b];
            if (lane == 31) *reinterpret_cast<uint32_t*>(stg + b * 528 + 512) = ov;
            uint32_t m0 = 0, m1 = 0;
#pragma unroll
            for (int i = 1; i < 16; i += 2) {
                auto win = [&](int n) -> uint32_t {
                    return (n & 3) ? __funnelshift_r(w[n >> 2], w[(n >> 2) + 1], 8 * (n & 3)) : w[n >> 2];
                };
                const uint32_t mid = win(i), a = win(i - 1), bb = win(i + 3);
                const uint32_t word = lds(base + (((mid * kPairMul) >> shift) << 2));
                uint32_t& m = i < 8 ? m0 : m1;
                m = __funnelshift_l(__funnelshift_l(0u, word, a), m, 1);
                m = __funnelshift_l(__funnelshift_l(0u, word, bb), m, 1);
            }
            masks[b] = (m0 << 8) | m1; // start j at bit 15 - j
            packed |= uint32_t(__popc(masks[b])) << (8 * b);
        }
        if (__any_sync(0xFFFFFFFFu, packed)) {
            uint32_t incl = packed;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= uint32_t(d)) incl += u;
            }
            const uint32_t totp = __shfl_sync(0xFFFFFFFFu, incl, 31);
            const uint32_t ex = incl - packed;
            uint32_t bstart = 0;
#pragma unroll
            for (int b = 0; b < B; ++b) {
                uint32_t at = bstart + ((ex >> (8 * b)) & 0xFF);
                for (uint32_t cm = masks[b]; cm; cm &= cm - 1)
                    q[at++] = uint16_t(b * 528 + 16 * lane + 15 - (__ffs(cm) - 1));
                bstart += (totp >> (8 * b)) & 0xFF;
            }
            __syncwarp();
            const uint32_t tot = bstart;
            uint32_t keep_n = 0;
            for (uint32_t r0 = 0; r0 < tot; r0 += 32) {
                bool keep = false;
                if (r0 + lane < tot) {
                    const uint32_t off = q[r0 + lane];
                    const uint32_t* wp = reinterpret_cast<const uint32_t*>(stg + (off & ~3u));
                    const uint32_t y = __funnelshift_r(wp[0], wp[1], 8 * off);
                    const bool odd = off & 1;
                    const uint32_t mid = odd ? y >> 8 : y, amt = odd ? y : y >> 24;
                    const uint32_t word = lds(base + (((mid * kPairMul) >> shift) << 2));
                    keep = int32_t(word << (amt & 31)) < 0;
                }
                keep_n += __popc(__ballot_sync(0xFFFFFFFFu, keep));
            }
            count += lane == 0 ? keep_n : 0;
        }
        __syncwarp();
    }
    for (int d = 16; d; d >>= 1) count += __shfl_xor_sync(0xFFFFFFFFu, count, d);
    if (lane == 0) atomicAdd(out, count);
}

template <int WARPS>
void run_batch(const uint4* d_text, uint64_t n16, const uint32_t* d_tab, uint32_t wb)
{
    unsigned long long* d_out;
    cudaMalloc(&d_out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = (size_t(4) << wb) + WARPS * (4 * 528 + 2048);
    cudaFuncSetAttribute(filt_batch<WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    float best = 1e9;
    unsigned long long cnt = 0;
    for (int it = 0; it < 8; ++it) {
        cudaMemset(d_out, 0, 8);
        cudaEventRecord(e0);
        filt_batch<WARPS><<<sms, WARPS * 32, smem>>>(d_text, n16, d_tab, wb, d_out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 2 && ms < best) best = ms;
        cudaMemcpy(&cnt, d_out, 8, cudaMemcpyDeviceToHost);
    }
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, filt_batch<WARPS>);
    printf("batch4 warps=%d regs=%d: %.3f ms  %.1f GB/s  survivors=%llu (%.4f%%)  err=%s\n", WARPS, fa.numRegs, best,
           n16 * 16 / best / 1e6, cnt, 100.0 * cnt / (n16 * 16.0), cudaGetErrorString(cudaGetLastError()));
    cudaFree(d_out);
}

int main(int argc, char** argv)
{
    const uint64_t bytes = 1ull << 30;
    const int npat = argc > 1 ? atoi(argv[1]) : 20000;
    const uint32_t wb = 15;
    std::vector<uint32_t> tab(1u << wb, 0);
    uint64_t x = 12345;
    for (int p = 0; p < npat; ++p) {
        x ^= x << 13, x ^= x >> 7, x ^= x << 17;
        const uint32_t g = uint32_t(x);
        tab[pair_word(g >> 8, wb)] |= 0x80000000u >> (g & 31);
        tab[pair_word(g & 0xFFFFFF, wb)] |= 0x80000000u >> ((g >> 24) & 31);
    }
    uint4* d_text;
    uint32_t* d_tab;
    cudaMalloc(&d_text, bytes + 64);
    cudaMalloc(&d_tab, tab.size() * 4);
    cudaMemcpy(d_tab, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice);
    fill<<<1024, 256>>>(d_text, bytes / 16, 7);
    cudaDeviceSynchronize();
    run_batch<16>(d_text, bytes / 16, d_tab, wb);
    run_batch<24>(d_text, bytes / 16, d_tab, wb);
    run_batch<32>(d_text, bytes / 16, d_tab, wb);
    for (int l2 = 0; l2 < 2; ++l2) {
        run<8>(d_text, bytes / 16, d_tab, wb, l2);
        run<16>(d_text, bytes / 16, d_tab, wb, l2);
        run<24>(d_text, bytes / 16, d_tab, wb, l2);
        run<32>(d_text, bytes / 16, d_tab, wb, l2);
    }
    return 0;
}

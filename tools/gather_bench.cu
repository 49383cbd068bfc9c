// Micro-benchmark of the access pattern that bounds k_slice_tile: 32 B (one sector) gathers
// from an L2-resident table T[N] (N = 1M -> 32 MB) at indices streamed from HBM, OR-reduced.
// Prints the achieved gather rate (sectors/s, GB/s of 32 B sectors) for several shapes, so
// the tile kernel's sweep can be compared with what the L2 delivers for this pattern.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>

template <int UNROLL, bool PAIR>
__global__ void __launch_bounds__(256) k_gather(const uint32_t *__restrict__ idx, const uint4 *__restrict__ T, uint64_t E,
                                                uint32_t *__restrict__ out) {
    // PAIR: a lane pair reads the two 16 B halves of one 32 B row (as k_slice_tile);
    // else one lane reads the whole 32 B row (two 16 B loads)
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint4 acc = make_uint4(0, 0, 0, 0);
    if (PAIR) {
        const uint64_t pr = tid >> 1, npr = nthr >> 1;
        const uint32_t half = tid & 1;
        uint64_t e = pr;
        for (; e + (UNROLL - 1) * npr < E; e += UNROLL * npr) {
            uint32_t y[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) y[u] = __ldg(idx + e + u * npr);
            uint4 v[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) v[u] = __ldg(T + 2ull * y[u] + half);
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) { acc.x |= v[u].x; acc.y |= v[u].y; acc.z |= v[u].z; acc.w |= v[u].w; }
        }
    } else {
        uint64_t e = tid;
        for (; e + (UNROLL - 1) * nthr < E; e += UNROLL * nthr) {
            uint32_t y[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) y[u] = __ldg(idx + e + u * nthr);
            uint4 v[2 * UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) { v[2 * u] = __ldg(T + 2ull * y[u]); v[2 * u + 1] = __ldg(T + 2ull * y[u] + 1); }
#pragma unroll
            for (int u = 0; u < 2 * UNROLL; ++u) { acc.x |= v[u].x; acc.y |= v[u].y; acc.z |= v[u].z; acc.w |= v[u].w; }
        }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[0] = 1;
}


// QUAD: a lane quad reads the four 16 B quarters of one 64 B record (two packs' 32 B T rows
// interleaved per individual): the 2-pack sweep's access pattern, 64 B per gather
template <int UNROLL>
__global__ void __launch_bounds__(256) k_gather64(const uint32_t *__restrict__ idx, const uint4 *__restrict__ T, uint64_t E,
                                                  uint32_t *__restrict__ out) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint64_t pr = tid >> 2, npr = nthr >> 2;
    const uint32_t q = tid & 3;
    uint64_t e = pr;
    for (; e + (UNROLL - 1) * npr < E; e += UNROLL * npr) {
        uint32_t y[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) y[u] = __ldg(idx + e + u * npr);
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = __ldg(T + 4ull * y[u] + q);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) { acc.x |= v[u].x; acc.y |= v[u].y; acc.z |= v[u].z; acc.w |= v[u].w; }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[0] = 1;
}

template <int U>
void run64(const char *name, const uint32_t *idx, const uint4 *T, uint64_t E, uint32_t *out, int blocks_per_sm, int sms) {
    const int grid = blocks_per_sm * sms;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) k_gather64<U><<<grid, 256>>>(idx, T, E, out);
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) k_gather64<U><<<grid, 256>>>(idx, T, E, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double s = ms / 1e3 / reps;
    printf("{\"shape\": \"%s\", \"bytes_per_gather\": 64, \"unroll\": %d, \"ctas_per_sm\": %d, \"us\": %.1f, "
           "\"ggathers_per_s\": %.1f, \"gather_gbs\": %.0f}\n", name, U, blocks_per_sm, s * 1e6, E / s / 1e9, 64.0 * E / s / 1e9);
}

template <int U, bool P>
void run(const char *name, const uint32_t *idx, const uint4 *T, uint64_t E, uint32_t *out, int blocks_per_sm, int sms,
         int smem = 0) {
    const int grid = blocks_per_sm * sms;
    if (smem) {
        cudaFuncSetAttribute(k_gather<U, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_gather<U, P>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) k_gather<U, P><<<grid, 256, smem>>>(idx, T, E, out);
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) k_gather<U, P><<<grid, 256, smem>>>(idx, T, E, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double s = ms / 1e3 / reps;
    printf("{\"shape\": \"%s\", \"unroll\": %d, \"pair\": %d, \"ctas_per_sm\": %d, \"smem_per_cta\": %d, \"us\": %.1f, "
           "\"gsectors_per_s\": %.1f, \"gather_gbs\": %.0f, \"idx_gbs\": %.0f}\n",
           name, U, (int)P, blocks_per_sm, smem, s * 1e6, E / s / 1e9, 32.0 * E / s / 1e9, 4.0 * E / s / 1e9);
}

int main() {
    const uint32_t N = 1u << 20;
    const uint64_t E = 8ull << 20;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::vector<uint32_t> h(E);
    std::mt19937 rng(7);
    for (uint64_t e = 0; e < E; ++e) h[e] = rng() % N;
    uint32_t *idx, *out;
    uint4 *T;
    cudaMalloc(&idx, E * 4);
    cudaMalloc(&T, (size_t)N * 64);
    cudaMalloc(&out, 4);
    cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice);
    cudaMemset(T, 0x5a, (size_t)N * 64);
    run<4, true>("uniform", idx, T, E, out, 4, sms);
    run<8, true>("uniform", idx, T, E, out, 4, sms);
    run64<4>("uniform", idx, T, E, out, 4, sms);
    run64<8>("uniform", idx, T, E, out, 4, sms);
    run64<8>("uniform", idx, T, E, out, 8, sms);
    run<4, true>("uniform", idx, T, E, out, 4, sms, 38400);
    run<8, true>("uniform", idx, T, E, out, 4, sms);
    run<4, true>("uniform", idx, T, E, out, 8, sms);
    run<8, true>("uniform", idx, T, E, out, 8, sms);
    run<4, false>("uniform", idx, T, E, out, 4, sms);
    run<4, false>("uniform", idx, T, E, out, 8, sms);
    run<8, false>("uniform", idx, T, E, out, 8, sms);
    // skewed targets as in the C3/C4 generator: popularity ~ (rank+1)^-0.8 over a random
    // permutation (a few individuals receive a large share of all gathers)
    {
        std::vector<double> cdf(N);
        double acc = 0;
        for (uint32_t k = 0; k < N; ++k) { acc += std::pow(k + 1.0, -0.8); cdf[k] = acc; }
        std::vector<uint32_t> perm(N);
        for (uint32_t k = 0; k < N; ++k) perm[k] = k;
        std::shuffle(perm.begin(), perm.end(), rng);
        std::uniform_real_distribution<double> U(0, acc);
        std::vector<uint32_t> hs(E);
        for (uint64_t e = 0; e < E; ++e) hs[e] = perm[std::lower_bound(cdf.begin(), cdf.end(), U(rng)) - cdf.begin()];
        cudaMemcpy(idx, hs.data(), E * 4, cudaMemcpyHostToDevice);
        run<4, true>("skewed", idx, T, E, out, 4, sms);
        run<8, true>("skewed", idx, T, E, out, 4, sms);
        run64<4>("skewed", idx, T, E, out, 4, sms);
        run64<8>("skewed", idx, T, E, out, 4, sms);
        // the tile kernel's shared-memory footprint (4 x 37.5 KB per SM) leaves less L1
        run<4, true>("skewed", idx, T, E, out, 4, sms, 38400);
        run<4, true>("skewed", idx, T, E, out, 4, sms, 54000);
        cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice);
    }
    // sorted indices (best-case locality) for contrast
    std::sort(h.begin(), h.end());
    cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice);
    run<4, true>("sorted", idx, T, E, out, 8, sms);
    return 0;
}

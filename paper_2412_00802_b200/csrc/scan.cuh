// Device exclusive scan (u8 or u32 values -> u32 offsets), three launches, used by the
// device planner and the top-k selection.  Header-only: kernels are per translation unit.
#pragma once
#include "internal.h"

namespace hedl {
namespace scan_detail {
namespace {
constexpr uint32_t FULLM = 0xffffffffu;
template <class T>
__global__ void __launch_bounds__(1024) k_scan_block(const T *__restrict__ in, uint32_t n, uint32_t *out,
                                                     uint32_t *bsum) {
    __shared__ uint32_t ws[32];
    const uint32_t i = blockIdx.x * 1024 + threadIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t v = i < n ? (uint32_t)in[i] : 0u;
    uint32_t x = v;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULLM, x, d);
        if (lane >= (uint32_t)d) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t t = ws[lane];
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(FULLM, t, d);
            if (lane >= (uint32_t)d) t += y;
        }
        ws[lane] = t;
    }
    __syncthreads();
    const uint32_t excl = x - v + (wid ? ws[wid - 1] : 0u);
    if (i < n) out[i] = excl;
    if (threadIdx.x == 1023) bsum[blockIdx.x] = excl + v;
}

__global__ void __launch_bounds__(1024) k_scan_sums(uint32_t *bsum, uint32_t nb, uint32_t *total) {
    __shared__ uint32_t ws[32];
    __shared__ uint32_t carry;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < nb; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < nb ? bsum[i] : 0u;
        uint32_t x = v;
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(FULLM, x, d);
            if (lane >= (uint32_t)d) x += y;
        }
        if (lane == 31) ws[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t t = ws[lane];
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(FULLM, t, d);
                if (lane >= (uint32_t)d) t += y;
            }
            ws[lane] = t;
        }
        __syncthreads();
        const uint32_t excl = x - v + (wid ? ws[wid - 1] : 0u) + carry;
        if (i < nb) bsum[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(1024) k_scan_add(uint32_t *out, uint32_t n, const uint32_t *__restrict__ bsum) {
    const uint32_t i = blockIdx.x * 1024 + threadIdx.x;
    if (i < n) out[i] += bsum[blockIdx.x];
}

inline uint32_t nblk(uint64_t n, uint32_t t) { return (uint32_t)((n + t - 1) / t); }
}  // namespace
}  // namespace scan_detail

// exclusive scan of n values at `in` into `out`; the total lands in *total (device)
template <class T>
inline void scan(cudaStream_t s, const T *in, uint32_t n, uint32_t *out, uint32_t *bsum, uint32_t *total) {
    const uint32_t nb = std::max<uint32_t>(1, scan_detail::nblk(n, 1024));
    if (n) scan_detail::k_scan_block<T><<<nb, 1024, 0, s>>>(in, n, out, bsum);
    else cudaMemsetAsync(bsum, 0, 4, s);
    scan_detail::k_scan_sums<<<1, 1024, 0, s>>>(bsum, n ? nb : 1, total);
    if (n) scan_detail::k_scan_add<<<nb, 1024, 0, s>>>(out, n, bsum);
    count_launch();
    count_launch();
    count_launch();
}

}  // namespace hedl

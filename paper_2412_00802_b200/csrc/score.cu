// hedl_score_topk: scores of evaluated hypotheses and the k best on the device (SURVEY
// 8(f) NEXT-3: "feeds a learner with on-device top-k"; score definitions: reading Q14).
//
// One score kernel (float64, the Q14 formulas), then an exact top-k selection without a
// full sort: scores in [0, 1] are non-negative doubles, whose bit patterns order like the
// values, so an 8-pass radix select over the 64-bit keys finds the k-th largest key T
// (per pass a shared-memory histogram of the current digit among the keys matching the
// prefix so far, and a one-warp pick of the digit); then the keys above T plus the
// lowest-index keys equal to T (an index-order scan) are the top k, sorted by (score
// descending, index ascending) with a single-CTA bitonic sort in shared memory.
#include <algorithm>

#include "internal.h"
#include "scan.cuh"

using namespace hedl;

namespace {

struct SelState {
    unsigned long long prefix, mask;
    uint32_t kk;          // rank still to find among the keys matching the prefix
    uint32_t cnt_gt;      // keys strictly above T collected so far
    uint32_t hist[256];
};

__global__ void k_score(const hedl_counts *__restrict__ c, uint32_t n, uint32_t metric, double *scores,
                        unsigned long long *keys) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const hedl_counts x = c[i];
    const double tp = (double)x.tp, fp = (double)x.fp, fn = (double)x.fn, tn = (double)x.tn;
    double num, den;
    if (metric == HEDL_SCORE_ACCURACY) { num = tp + tn; den = tp + fp + fn + tn; }
    else { num = 2.0 * tp; den = 2.0 * tp + fp + fn; }
    const double s = den > 0.0 ? num / den : 0.0;
    if (scores) scores[i] = s;
    keys[i] = (unsigned long long)__double_as_longlong(s);
}

__global__ void k_radix_hist(const unsigned long long *__restrict__ keys, uint32_t n, SelState *st, uint32_t shift) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long prefix = st->prefix, mask = st->mask;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
        if ((k & mask) == prefix) atomicAdd(h + ((k >> shift) & 255u), 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(st->hist + threadIdx.x, h[threadIdx.x]);
}

__global__ void k_radix_pick(SelState *st, uint32_t shift) {
    if (threadIdx.x == 0) {
        uint32_t cum = 0;
        for (int d = 255; d >= 0; --d) {
            const uint32_t c = st->hist[d];
            if (cum + c >= st->kk) {
                st->prefix |= (unsigned long long)d << shift;
                st->mask |= 255ull << shift;
                st->kk -= cum;
                break;
            }
            cum += c;
        }
    }
    __syncthreads();
    st->hist[threadIdx.x] = 0;
}

__global__ void k_collect_gt(const unsigned long long *__restrict__ keys, uint32_t n, SelState *st, uint32_t *cand,
                             uint8_t *eq) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = keys[i], t = st->prefix;
    eq[i] = k == t;
    if (k > t) cand[atomicAdd(&st->cnt_gt, 1u)] = i;
}

__global__ void k_collect_eq(const uint8_t *__restrict__ eq, const uint32_t *__restrict__ rank, uint32_t n, const SelState *st,
                             uint32_t k, uint32_t *cand) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !eq[i]) return;
    const uint32_t r = rank[i];
    if (r < st->kk) cand[k - st->kk + r] = i;
}

// single CTA: bitonic sort of the k candidates by (key descending, index ascending)
__global__ void __launch_bounds__(1024) k_sort_topk(const uint32_t *__restrict__ cand, uint32_t k, uint32_t P,
                                                    const unsigned long long *__restrict__ keys, uint32_t *top_idx,
                                                    double *top_scores) {
    extern __shared__ unsigned long long sk[];
    uint32_t *si = (uint32_t *)(sk + P);
    for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
        if (t < k) { si[t] = cand[t]; sk[t] = keys[cand[t]]; }
        else { si[t] = 0xffffffffu; sk[t] = 0; }
    }
    __syncthreads();
    auto before = [&](uint32_t a, uint32_t b) {       // a sorts before b
        return sk[a] > sk[b] || (sk[a] == sk[b] && si[a] < si[b]);
    };
    for (uint32_t size = 2; size <= P; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
                const uint32_t u = t ^ stride;
                if (u > t) {
                    const bool up = (t & size) == 0;        // this run sorts in the "before" order
                    const bool swap = up ? before(u, t) : before(t, u);
                    if (swap) {
                        const unsigned long long tk = sk[t]; sk[t] = sk[u]; sk[u] = tk;
                        const uint32_t ti = si[t]; si[t] = si[u]; si[u] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t t = threadIdx.x; t < k; t += blockDim.x) {
        if (top_idx) top_idx[t] = si[t];
        if (top_scores) top_scores[t] = __longlong_as_double((long long)sk[t]);
    }
}

inline uint32_t nblk(uint64_t n, uint32_t t) { return (uint32_t)((n + t - 1) / t); }

}  // namespace

extern "C" hedl_status hedl_score_topk(const hedl_counts *counts, uint32_t n, uint32_t metric, uint32_t k,
                                       double *scores, uint32_t *top_idx, double *top_scores, int device,
                                       void *stream) {
    if (metric > HEDL_SCORE_F1) return fail(HEDL_ERR_INVALID_ARG, "unknown metric");
    if (k > n || k > kTopKMax) return fail(HEDL_ERR_INVALID_ARG, "k must be <= n and <= 4096");
    if (n && !counts) return fail(HEDL_ERR_INVALID_ARG, "null counts");
    if (k && !top_idx && !top_scores) return fail(HEDL_ERR_INVALID_ARG, "k > 0 needs top_idx or top_scores");
    if (!n) return HEDL_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != device && cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return fail(HEDL_ERR_UNSUPPORTED, "no such device"); }
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};
    cudaStream_t s = (cudaStream_t)stream;
    {   // keep freed stream-ordered scratch mapped (the default release threshold of 0 would
        // hand it back to the OS at every synchronisation and re-map it on the next call)
        static std::mutex mu;
        static uint64_t done_mask = 0;
        std::lock_guard<std::mutex> lk(mu);
        if (device < 64 && !(done_mask >> device & 1)) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
                uint64_t thr = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            cudaGetLastError();
            done_mask |= 1ull << device;
        }
    }
    // stream-ordered scratch: keys, eq flags, ranks, candidates, block sums, state
    Carver c;
    c.take<unsigned long long>(n);
    c.take<uint8_t>(n);
    c.take<uint32_t>(n);
    c.take<uint32_t>(std::max<uint32_t>(k, 1));
    c.take<uint32_t>(nblk(n, 1024) + 1);
    c.take<uint32_t>(8);
    c.take<SelState>(1);
    void *blk = nullptr;
    // the caller's allocator when installed (hedl_set_allocator), else the stream-ordered pool
    cudaError_t e = dev_alloc_installed() ? dev_malloc(&blk, c.off, s) : cudaMallocAsync(&blk, c.off, s);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(HEDL_ERR_OOM, "top-k scratch"); }
    Carver d{(char *)blk, 0};
    unsigned long long *keys = d.take<unsigned long long>(n);
    uint8_t *eq = d.take<uint8_t>(n);
    uint32_t *rank = d.take<uint32_t>(n);
    uint32_t *cand = d.take<uint32_t>(std::max<uint32_t>(k, 1));
    uint32_t *bsum = d.take<uint32_t>(nblk(n, 1024) + 1);
    uint32_t *tot = d.take<uint32_t>(8);
    SelState *st = d.take<SelState>(1);
    k_score<<<nblk(n, 256), 256, 0, s>>>(counts, n, metric, scores, keys);
    count_launch();
    if (k) {
        SelState init{};
        init.kk = k;
        cudaMemcpyAsync(st, &init, sizeof(init), cudaMemcpyHostToDevice, s);
        const uint32_t gx = std::min<uint32_t>(nblk(n, 256), 1184);
        for (int shift = 56; shift >= 0; shift -= 8) {
            k_radix_hist<<<gx, 256, 0, s>>>(keys, n, st, (uint32_t)shift);
            k_radix_pick<<<1, 256, 0, s>>>(st, (uint32_t)shift);
            count_launch();
            count_launch();
        }
        k_collect_gt<<<nblk(n, 256), 256, 0, s>>>(keys, n, st, cand, eq);
        scan(s, eq, n, rank, bsum, tot);
        k_collect_eq<<<nblk(n, 256), 256, 0, s>>>(eq, rank, n, st, k, cand);
        uint32_t P = 1;
        while (P < k) P <<= 1;
        const size_t smem = (size_t)P * 12;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_sort_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_sort_topk<<<1, 1024, smem, s>>>(cand, k, P, keys, top_idx, top_scores);
        for (int q = 0; q < 3; ++q) count_launch();
    }
    if (dev_alloc_installed()) dev_free(blk, s);
    else cudaFreeAsync(blk, s);
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(HEDL_ERR_CUDA, std::string("score_topk: ") + cudaGetErrorString(e));
    return HEDL_OK;
}

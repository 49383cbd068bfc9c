// Latency path of hedl_eval_one (SURVEY 8(a) "small N": a single-launch bytecode
// interpreter).  The root's canonical sub-DAG travels as a kernel parameter (no H2D copy)
// and is walked in topological order with every intermediate row in shared memory; the
// four counts are written straight into mapped pinned host memory -- one launch and one
// stream sync per hypothesis.  Small KBs run on one CTA of 1024 threads (k_interp); KBs of
// kInterpClusterMinW4 words or more on a cluster of kInterpCl CTAs that split every row's
// words and complete the rows restrictions read through distributed shared memory
// (k_interp_cl).  Semantics are those of the batch kernels (kernels.cu): the same
// count-with-saturation predicates (Algs. 4, 6, 7-8), complement masks (Alg. 2), float32
// closed-interval ranges (Alg. 10, Q9) and Alg. 15 coverage.
#include <cooperative_groups.h>

#include "interp.h"

namespace cg = cooperative_groups;

namespace hedl {

namespace {
constexpr uint32_t FULL = 0xffffffffu;

__device__ __forceinline__ bool pred_ok(uint32_t pred, uint32_t cnt, uint32_t n) {
    switch (pred) {
    case P_GE: return cnt >= n;
    case P_LE: return cnt <= n;
    case P_EQ: return cnt == n;
    default: return cnt > 0 && cnt <= n;
    }
}

struct IKb {
    uint32_t N, W, W4;
    const uint32_t *concepts, *ones, *pos, *neg;
    const uint32_t *const *row_ptr;   // per direction (device array of pointers)
    const uint32_t *const *col;
    const uint32_t *const *drow;      // per data property
    const float *const *dval;
};

__device__ __forceinline__ const uint32_t *operand(const IKb &kb, const uint32_t *smem, uint32_t ref) {
    const uint32_t id = ref >> 3;
    switch ((ref >> 1) & 3u) {
    case RT_NODE: return smem + (size_t)id * kb.W4;
    case RT_ATOM: return kb.concepts + (size_t)id * kb.W4;
    default: return kb.ones;
    }
}

__global__ void __launch_bounds__(1024) k_interp(IKb kb, InterpProg prog, hedl_counts *counts, uint32_t *out_bits) {
    extern __shared__ uint32_t srows[];
    __shared__ uint32_t s_red[2][32];
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    for (uint32_t i = 0; i < prog.n_nodes; ++i) {
        const InterpNode nd = prog.nodes[i];
        const uint32_t kind = nd.kind & 0x7fu;
        uint32_t *out = srows + (size_t)i * kb.W4;
        if (kind == NK_AND || kind == NK_OR) {
            for (uint32_t w = tid; w < kb.W4; w += blockDim.x) {
                uint32_t acc = kind == NK_OR ? 0u : FULL;
                for (uint32_t q = 0; q < nd.op_count; ++q) {
                    const uint32_t r = prog.ops[nd.op_begin + q];
                    const uint32_t v = operand(kb, srows, r)[w] ^ ((r & 1u) ? FULL : 0u);
                    acc = kind == NK_OR ? (acc | v) : (acc & v);
                }
                if (w >= kb.W) acc = 0;
                else if (w == kb.W - 1 && (kb.N & 31)) acc &= (1u << (kb.N & 31)) - 1u;
                out[w] = acc;
            }
        } else if (kind == NK_RESTRICT) {
            const uint32_t r = prog.ops[nd.op_begin];
            const uint32_t *child = operand(kb, srows, r);
            const uint32_t cm = (r & 1u) ? FULL : 0u;
            const uint32_t *rp = kb.row_ptr[nd.dir], *cl = kb.col[nd.dir];
            // x = base + tid, the warp's 32 consecutive rows make one output word
            for (uint32_t base = 0; base < kb.W4 * 32; base += blockDim.x) {
                const uint32_t x = base + tid;
                bool res = false;
                if (x < kb.N) {
                    const uint32_t a = __ldg(rp + x), b = __ldg(rp + x + 1);
                    uint32_t cnt = 0;
                    for (uint32_t e = a; e < b && cnt < nd.sat; ++e) {
                        const uint32_t y = __ldg(cl + e);
                        cnt += ((child[y >> 5] ^ cm) >> (y & 31)) & 1u;
                    }
                    res = pred_ok(nd.pred, min(cnt, nd.sat), nd.n);
                }
                const uint32_t word = __ballot_sync(FULL, res);
                if (lane == 0 && (x >> 5) < kb.W4) out[x >> 5] = word;
            }
        } else {
            const uint32_t *rp = kb.drow[nd.dir];
            const float *val = kb.dval[nd.dir];
            for (uint32_t base = 0; base < kb.W4 * 32; base += blockDim.x) {
                const uint32_t x = base + tid;
                bool res = false;
                if (x < kb.N) {
                    uint32_t lo = __ldg(rp + x), hi = __ldg(rp + x + 1);
                    const uint32_t end = hi;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (__ldg(val + mid) < nd.lo) lo = mid + 1; else hi = mid;
                    }
                    res = lo < end && __ldg(val + lo) <= nd.hi;
                }
                const uint32_t word = __ballot_sync(FULL, res);
                if (lane == 0 && (x >> 5) < kb.W4) out[x >> 5] = word;
            }
        }
        __syncthreads();
    }
    // Alg. 15 coverage of the root (the last node), one reduction, counts to mapped host memory
    const uint32_t *root = srows + (size_t)(prog.n_nodes - 1) * kb.W4;
    uint32_t tp = 0, fp = 0;
    for (uint32_t w = tid; w < kb.W; w += blockDim.x) {
        const uint32_t h = root[w];
        tp += __popc(h & __ldg(kb.pos + w));
        fp += __popc(h & __ldg(kb.neg + w));
        if (out_bits) out_bits[w] = h;
    }
    tp = __reduce_add_sync(FULL, tp);
    fp = __reduce_add_sync(FULL, fp);
    if (lane == 0) { s_red[0][tid >> 5] = tp; s_red[1][tid >> 5] = fp; }
    __syncthreads();
    if (tid < 32) {
        uint32_t a = tid < (blockDim.x >> 5) ? s_red[0][tid] : 0u, b = tid < (blockDim.x >> 5) ? s_red[1][tid] : 0u;
        a = __reduce_add_sync(FULL, a);
        b = __reduce_add_sync(FULL, b);
        if (tid == 0) {
            counts->tp = a;
            counts->fp = b;
            counts->fn = prog.npos - a;
            counts->tn = prog.nneg - b;
            __threadfence_system();                       // counts (and the row) before the flag
            *(volatile unsigned long long *)&counts[1].tp = prog.seq;
        }
    }
}

// Cluster interpreter (KBs of >= kInterpClusterMinW4 words): the same program over kInterpCl
// CTAs of one thread-block cluster.  CTA r computes its word slice [r*WC, (r+1)*WC) of every
// node; rows read at arbitrary individuals (restriction fillers, InterpNode kind bit 7) are
// completed after their node by copying the other CTAs' slices out of their shared memory
// (distributed shared memory, cluster barrier), everything else stays slice-local.  Counts:
// each CTA's slice of the root, summed by rank 0 through DSMEM.
__global__ void __cluster_dims__(kInterpCl, 1, 1) __launch_bounds__(1024)
    k_interp_cl(IKb kb, InterpProg prog, hedl_counts *counts, uint32_t *out_bits) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ uint32_t srows[];
    __shared__ uint32_t s_red[2][32];
    __shared__ unsigned long long s_tp, s_fp;
    const uint32_t tid = threadIdx.x, lane = tid & 31, r = cl.block_rank();
    const uint32_t WC = (kb.W4 + 4 * kInterpCl - 1) / (4 * kInterpCl) * 4;
    const uint32_t wlo = min(kb.W4, r * WC), whi = min(kb.W4, (r + 1) * WC);
    for (uint32_t i = 0; i < prog.n_nodes; ++i) {
        const InterpNode nd = prog.nodes[i];
        const uint32_t kind = nd.kind & 0x7fu;
        uint32_t *out = srows + (size_t)i * kb.W4;
        if (kind == NK_AND || kind == NK_OR) {
            for (uint32_t w = wlo + tid; w < whi; w += blockDim.x) {
                uint32_t acc = kind == NK_OR ? 0u : FULL;
                for (uint32_t q = 0; q < nd.op_count; ++q) {
                    const uint32_t rr = prog.ops[nd.op_begin + q];
                    const uint32_t v = operand(kb, srows, rr)[w] ^ ((rr & 1u) ? FULL : 0u);
                    acc = kind == NK_OR ? (acc | v) : (acc & v);
                }
                if (w >= kb.W) acc = 0;
                else if (w == kb.W - 1 && (kb.N & 31)) acc &= (1u << (kb.N & 31)) - 1u;
                out[w] = acc;
            }
        } else if (kind == NK_RESTRICT) {
            const uint32_t rr = prog.ops[nd.op_begin];
            const uint32_t *child = operand(kb, srows, rr);
            const uint32_t cm = (rr & 1u) ? FULL : 0u;
            const uint32_t *rp = kb.row_ptr[nd.dir], *clp = kb.col[nd.dir];
            for (uint32_t base = wlo * 32; base < whi * 32; base += blockDim.x) {
                const uint32_t x = base + tid;
                bool res = false;
                if (x < kb.N && x < whi * 32) {
                    const uint32_t a = __ldg(rp + x), b = __ldg(rp + x + 1);
                    uint32_t cnt = 0;
                    for (uint32_t e = a; e < b && cnt < nd.sat; ++e) {
                        const uint32_t y = __ldg(clp + e);
                        cnt += ((child[y >> 5] ^ cm) >> (y & 31)) & 1u;
                    }
                    res = pred_ok(nd.pred, min(cnt, nd.sat), nd.n);
                }
                const uint32_t word = __ballot_sync(FULL, res);
                if (lane == 0 && (x >> 5) < whi) out[x >> 5] = word;
            }
        } else {
            const uint32_t *rp = kb.drow[nd.dir];
            const float *val = kb.dval[nd.dir];
            for (uint32_t base = wlo * 32; base < whi * 32; base += blockDim.x) {
                const uint32_t x = base + tid;
                bool res = false;
                if (x < kb.N && x < whi * 32) {
                    uint32_t lo = __ldg(rp + x), hi = __ldg(rp + x + 1);
                    const uint32_t end = hi;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (__ldg(val + mid) < nd.lo) lo = mid + 1; else hi = mid;
                    }
                    res = lo < end && __ldg(val + lo) <= nd.hi;
                }
                const uint32_t word = __ballot_sync(FULL, res);
                if (lane == 0 && (x >> 5) < whi) out[x >> 5] = word;
            }
        }
        if (nd.kind & 0x80u) {                            // a restriction reads this row anywhere
            cl.sync();                                    // every slice of row i is complete
            for (uint32_t q = 1; q < kInterpCl; ++q) {
                const uint32_t src = (r + q) % kInterpCl;
                const uint32_t *rem = cl.map_shared_rank(srows, src) + (size_t)i * kb.W4;
                const uint32_t a = min(kb.W4, src * WC), b = min(kb.W4, (src + 1) * WC);
                for (uint32_t w = a + tid; w < b; w += blockDim.x) out[w] = rem[w];
            }
        }
        __syncthreads();
    }
    // Alg. 15 coverage of the root over this CTA's slice; rank 0 sums the slices
    const uint32_t *root = srows + (size_t)(prog.n_nodes - 1) * kb.W4;
    uint32_t tp = 0, fp = 0;
    for (uint32_t w = wlo + tid; w < min(whi, kb.W); w += blockDim.x) {
        const uint32_t h = root[w];
        tp += __popc(h & __ldg(kb.pos + w));
        fp += __popc(h & __ldg(kb.neg + w));
        if (out_bits) out_bits[w] = h;
    }
    tp = __reduce_add_sync(FULL, tp);
    fp = __reduce_add_sync(FULL, fp);
    if (lane == 0) { s_red[0][tid >> 5] = tp; s_red[1][tid >> 5] = fp; }
    __syncthreads();
    if (tid < 32) {
        uint32_t a = tid < (blockDim.x >> 5) ? s_red[0][tid] : 0u, b = tid < (blockDim.x >> 5) ? s_red[1][tid] : 0u;
        a = __reduce_add_sync(FULL, a);
        b = __reduce_add_sync(FULL, b);
        if (tid == 0) { s_tp = a; s_fp = b; }
    }
    cl.sync();
    if (r == 0 && tid == 0) {
        unsigned long long a = 0, b = 0;
        for (uint32_t q = 0; q < kInterpCl; ++q) {
            a += *cl.map_shared_rank(&s_tp, q);
            b += *cl.map_shared_rank(&s_fp, q);
        }
        counts->tp = a;
        counts->fp = b;
        counts->fn = prog.npos - a;
        counts->tn = prog.nneg - b;
        __threadfence_system();                           // counts (and the row) before the flag
        *(volatile unsigned long long *)&counts[1].tp = prog.seq;
    }
    cl.sync();                                            // keep shared memory alive for rank 0
}
}  // namespace

size_t interp_smem_limit() { return 200u * 1024u; }

hedl_status interp_prepare(hedl_kb *kb) {
    // device arrays of per-direction / per-property pointers for the interpreter
    if (kb->interp_ptrs || !kb->dirs.size() && !kb->data.size()) return HEDL_OK;
    std::vector<const void *> h;
    for (auto &d : kb->dirs) h.push_back(d.row_ptr);
    for (auto &d : kb->dirs) h.push_back(d.col);
    for (auto &d : kb->data) h.push_back(d.row_ptr);
    for (auto &d : kb->data) h.push_back(d.val);
    void *p = nullptr;
    if (dev_malloc(&p, h.size() * sizeof(void *)) != cudaSuccess) { cudaGetLastError(); return fail(HEDL_ERR_OOM, "interp pointers"); }
    kb->allocs.push_back(p);
    if (cudaMemcpy(p, h.data(), h.size() * sizeof(void *), cudaMemcpyHostToDevice) != cudaSuccess)
        return cuda_fail(kb, cudaGetLastError(), "interp pointers");
    kb->interp_ptrs = (const void **)p;
    return HEDL_OK;
}

hedl_status interp_launch(const hedl_kb *kb, const InterpProg &prog, hedl_counts *counts_mapped, uint32_t *out_bits,
                          cudaStream_t s) {
    const size_t R = kb->dirs.size(), D = kb->data.size();
    const void *const *pp = (const void *const *)kb->interp_ptrs;
    IKb ik{kb->N, kb->W, kb->W4, kb->concepts, kb->ones, kb->pos, kb->neg,
           (const uint32_t *const *)pp, (const uint32_t *const *)(pp + R),
           (const uint32_t *const *)(pp + 2 * R), (const float *const *)(pp + 2 * R + D)};
    const size_t smem = (size_t)prog.n_nodes * kb->W4 * 4;
    static std::once_flag attr[kMaxDevices];
    once_per_device(attr, [] {
        cudaFuncSetAttribute(k_interp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)interp_smem_limit());
        cudaFuncSetAttribute(k_interp_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)interp_smem_limit());
    });
    prof_begin(s, KC_INTERP);
    if (kb->W4 >= kInterpClusterMinW4) k_interp_cl<<<kInterpCl, 1024, smem, s>>>(ik, prog, counts_mapped, out_bits);
    else k_interp<<<1, 1024, smem, s>>>(ik, prog, counts_mapped, out_bits);
    count_launch();
    prof_end(s, KC_INTERP, 0, prog.n_nodes);
    HEDL_CUDA(kb, cudaGetLastError());
    return HEDL_OK;
}

}  // namespace hedl

// Device planner: the evaluation plan of a device-compiled program built
// on the GPU ("each GPU generates its evaluation plans
// ... with minimal to no CPU intervention").
//
// The same plan as the host planner (exec.cu, fill_chunk) for a single chunk: live
// nodes, one count slot per distinct root node, row demands (full rows only for nodes
// another node reads in full, example-projected rows for the rest), launch groups by
// (level, kind, direction, lane-pack class, demand), descriptors with final device
// addresses.  Every per-node step is a kernel; the host reads back one small table
// (per-group counts, a few KB) to size the buffers and issue the launches.
#include <algorithm>

#include "exec.h"
#include "scan.cuh"
#include "slice.h"

using namespace hedl;

namespace {

constexpr uint32_t FULLM = 0xffffffffu;
constexpr uint8_t NK_DEAD_D = 0xff;
constexpr uint32_t kKinds = 4;          // AND/OR, RESTRICT, DRANGE, STRING
constexpr uint32_t kSub = 6;            // class (3) x demand split (2)
constexpr uint32_t kMaxBuckets = 1u << 22;

__device__ __forceinline__ uint32_t d_slice_class(uint32_t n, uint32_t sat) {
    if (sat <= 1) return 0;
    if (n <= 30 && sat <= 31) return 1;
    return 2;
}
__device__ __forceinline__ bool d_isnode(uint32_t r) { return ((r >> 1) & 3u) == RT_NODE; }

inline uint32_t nblk(uint64_t n, uint32_t t) { return (uint32_t)((n + t - 1) / t); }

// ---- live nodes, level lists -------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_dp_level_hist(const CNode *__restrict__ nodes, uint32_t nn, uint32_t *hist,
                                                        uint32_t nkeys) {
    extern __shared__ uint32_t sh[];
    for (uint32_t k = threadIdx.x; k < nkeys; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x)
        if (nodes[i].kind != NK_DEAD_D) atomicAdd(sh + nodes[i].level, 1u);
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < nkeys; k += blockDim.x)
        if (sh[k]) atomicAdd(hist + k, sh[k]);
}
__global__ void __launch_bounds__(1024) k_dp_level_scatter(const CNode *__restrict__ nodes, uint32_t nn, uint32_t *cursor,
                                                           uint32_t *list, uint32_t nkeys) {
    extern __shared__ uint32_t sh[];
    for (uint32_t k = threadIdx.x; k < 2 * nkeys; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t key = 0, r = 0;
    const bool on = i < nn && nodes[i].kind != NK_DEAD_D;
    if (on) {
        key = nodes[i].level;
        r = atomicAdd(sh + key, 1u);
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < nkeys; k += blockDim.x)
        if (sh[k]) sh[nkeys + k] = atomicAdd(cursor + k, sh[k]);
    __syncthreads();
    if (on) list[sh[nkeys + key] + r] = i;
}

__global__ void k_dp_init(const CNode *__restrict__ nodes, uint32_t nn, bool all, uint8_t *live, uint8_t *isroot,
                          uint8_t *nfull, uint8_t *nproj) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    live[i] = all && nodes[i].kind != NK_DEAD_D;
    isroot[i] = 0;
    nfull[i] = 0;
    nproj[i] = 0;
}

__global__ void k_dp_roots(const uint32_t *__restrict__ root_node, uint32_t r0, uint32_t r1, bool bits, uint8_t *live,
                           uint8_t *isroot, uint8_t *nfull) {
    const uint32_t r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r1) return;
    const uint32_t x = root_node[r];
    live[x] = 1;
    isroot[x] = 1;
    if (bits) nfull[x] = 1;
}

__global__ void k_dp_mark_down(const uint32_t *__restrict__ list, uint32_t m, const CNode *__restrict__ nodes,
                               const uint32_t *__restrict__ ops, uint8_t *live) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t i = list[t];
    if (!live[i]) return;
    const CNode n = nodes[i];
    for (uint32_t q = 0; q < n.op_count; ++q) {
        const uint32_t o = ops[n.op_begin + q];
        if (d_isnode(o)) live[o >> 3] = 1;
    }
}

// demands, consumers first (one level per launch, top down; within a level nodes are
// independent, concurrent stores of 1 to a shared operand flag are benign)
__global__ void k_dp_demand(const uint32_t *__restrict__ list, uint32_t m, const CNode *__restrict__ nodes,
                            const uint32_t *__restrict__ ops, const uint8_t *__restrict__ live, uint8_t *nfull,
                            uint8_t *nproj, uint8_t *pmode) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t i = list[t];
    if (!live[i]) return;
    const CNode n = nodes[i];
    const bool pm = (n.kind == NK_AND || n.kind == NK_OR) && !nfull[i];
    pmode[i] = pm;
    for (uint32_t q = 0; q < n.op_count; ++q) {
        const uint32_t o = ops[n.op_begin + q];
        if (!d_isnode(o)) continue;
        if (pm) nproj[o >> 3] = 1;
        else nfull[o >> 3] = 1;
    }
}

struct BucketGeom {
    uint32_t dirs, nbuckets;
};

__device__ __forceinline__ uint32_t d_bucket(const CNode &n, bool pmode, bool nfull, const BucketGeom &g,
                                             uint32_t *cls_out) {
    const uint32_t kc = (n.kind == NK_AND || n.kind == NK_OR) ? 0u : n.kind == NK_RESTRICT ? 1u : n.kind == NK_DRANGE ? 2u : 3u;
    uint32_t cls = 0, sub = 0;
    if (kc == 0) sub = pmode;
    else if (kc == 1) {
        cls = d_slice_class(n.n, n.sat);
        sub = cls < 2 && !nfull;
    }
    const uint32_t dir = kc == 0 ? 0u : n.dir;
    *cls_out = cls;
    return ((n.level * kKinds + kc) * g.dirs + dir) * kSub + cls * 2 + sub;
}

// per bucket: count, operands (boolean), rows written, coverage slots
__global__ void k_dp_bucket(const CNode *__restrict__ nodes, uint32_t nn, const uint8_t *__restrict__ live,
                            const uint8_t *__restrict__ pmode, const uint8_t *__restrict__ nfull,
                            const uint8_t *__restrict__ nproj, const uint8_t *__restrict__ isroot, BucketGeom g,
                            uint32_t *bucket, uint32_t *b_count, uint32_t *b_ops, uint32_t *b_outs, uint32_t *b_cov) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    uint32_t b = FULLM, ops = 0, outs = 0, cov = 0;
    if (i < nn && live[i]) {
        const CNode n = nodes[i];
        uint32_t cls;
        b = d_bucket(n, pmode[i], nfull[i], g, &cls);
        bucket[i] = b;
        const bool isbool = n.kind == NK_AND || n.kind == NK_OR;
        ops = isbool ? n.op_count : 0;
        outs = (isbool && pmode[i]) ? nproj[i] : nfull[i];
        cov = isroot[i];
    }
    // warp aggregation by bucket: one atomic per distinct bucket per warp
    const uint32_t peers = __match_any_sync(FULLM, b);
    const uint32_t leader = __ffs(peers) - 1;
    uint32_t s_ops = 0, s_outs = 0, s_cov = 0;
    for (uint32_t l = 0; l < 32; ++l) {
        const uint32_t a = __shfl_sync(FULLM, ops, l), o = __shfl_sync(FULLM, outs, l), c = __shfl_sync(FULLM, cov, l);
        if (peers & (1u << l)) { s_ops += a; s_outs += o; s_cov += c; }
    }
    if (b != FULLM && lane == leader) {
        atomicAdd(b_count + b, (uint32_t)__popc(peers));
        if (s_ops) atomicAdd(b_ops + b, s_ops);
        if (s_outs) atomicAdd(b_outs + b, s_outs);
        if (s_cov) atomicAdd(b_cov + b, s_cov);
    }
}

// desc position of every live node: first[bucket] + rank (warp-aggregated cursor)
__global__ void k_dp_scatter(uint32_t nn, const uint8_t *__restrict__ live, const uint32_t *__restrict__ bucket,
                             const uint32_t *__restrict__ first, uint32_t *cursor, uint32_t *dnode, uint32_t *rank_of) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t b = (i < nn && live[i]) ? bucket[i] : FULLM;
    const uint32_t peers = __match_any_sync(FULLM, b);
    const uint32_t leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (b != FULLM && lane == leader) base = atomicAdd(cursor + b, (uint32_t)__popc(peers));
    base = __shfl_sync(FULLM, base, leader);
    if (b == FULLM) return;
    const uint32_t r = base + __popc(peers & ((1u << lane) - 1u));
    const uint32_t pos = first[b] + r;
    dnode[pos] = i;
    rank_of[i] = r;
}

__global__ void k_dp_opc(const uint32_t *__restrict__ dnode, uint32_t nb, const CNode *__restrict__ nodes, uint32_t *opc) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nb) opc[t] = nodes[dnode[t]].op_count;
}

struct FillArgs {
    const CNode *nodes;
    const uint32_t *ops;
    const uint32_t *dnode, *rank_of, *opfirst, *slot, *pslot, *cover;
    const uint8_t *nfull, *nproj, *pmode, *isroot;
    uint32_t nb, nr, nd;                  // descriptor counts per type (bool, restrict, range)
    BoolDesc *bd;
    Operand *od;
    RestrictDesc *rd;
    DrangeDesc *dd;
    uint32_t *rows, *prows;
    const uint32_t *concepts, *ones, *pconcepts, *pones;
    uint32_t W4, MW4;
    uint32_t n_heavy[64];
};

__device__ __forceinline__ const uint32_t *d_ptr_of(const FillArgs &a, uint32_t r) {
    const uint32_t t = (r >> 1) & 3u, id = r >> 3;
    if (t == RT_NODE) return a.rows + (size_t)a.slot[id] * a.W4;
    if (t == RT_ATOM) return a.concepts + (size_t)id * a.W4;
    return a.ones;
}
__device__ __forceinline__ const uint32_t *d_pptr_of(const FillArgs &a, uint32_t r) {
    const uint32_t t = (r >> 1) & 3u, id = r >> 3;
    if (t == RT_NODE) return a.prows + (size_t)a.pslot[id] * a.MW4;
    if (t == RT_ATOM) return a.pconcepts + (size_t)id * a.MW4;
    return a.pones;
}

__global__ void k_dp_fill(FillArgs a) {
    const uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= a.nb + a.nr + a.nd) return;
    const uint32_t k = a.dnode[pos];
    const CNode n = a.nodes[k];
    uint32_t *out = a.nfull[k] ? a.rows + (size_t)a.slot[k] * a.W4 : nullptr;
    uint32_t *proj = a.nproj[k] ? a.prows + (size_t)a.pslot[k] * a.MW4 : nullptr;
    const int32_t cover = a.isroot[k] ? (int32_t)a.cover[k] : -1;
    if (pos < a.nb) {
        BoolDesc d;
        const bool pm = a.pmode[k];
        d.out = pm ? proj : out;
        d.proj = pm ? nullptr : proj;
        d.op_first = a.opfirst[pos];
        d.op_count = n.op_count;
        d.is_or = n.kind == NK_OR;
        d.cover = cover;
        for (uint32_t q = 0; q < n.op_count; ++q) {
            const uint32_t o = a.ops[n.op_begin + q];
            a.od[d.op_first + q] = Operand{pm ? d_pptr_of(a, o) : d_ptr_of(a, o), (o & 1u) ? 0xffffffffu : 0u, 0};
        }
        a.bd[pos] = d;
    } else if (pos < a.nb + a.nr) {
        const uint32_t c = a.ops[n.op_begin];
        RestrictDesc d;
        d.child = d_ptr_of(a, c);
        d.out = out;
        d.proj = proj;
        d.cmask = (c & 1u) ? 0xffffffffu : 0u;
        d.pred = n.pred;
        d.n = n.n;
        d.sat = n.sat;
        d.cover = cover;
        d.heavy_slot = a.rank_of[k] * a.n_heavy[n.dir & 63];
        d.op_first = d.op_n = 0;
        d.uout = nullptr;
        d.udirs = d.pad_ = 0;
        a.rd[pos - a.nb] = d;
    } else {
        DrangeDesc d;
        d.out = out;
        d.proj = proj;
        d.lo = n.lo;
        d.hi = n.hi;
        d.cover = cover;
        d.prop = n.dir;
        a.dd[pos - a.nb - a.nr] = d;
    }
}

__global__ void k_dp_root_tables(const uint32_t *__restrict__ root_node, uint32_t r0, uint32_t n,
                                 const uint32_t *__restrict__ cover, const uint32_t *__restrict__ slot, uint32_t *rows,
                                 uint32_t W4, uint32_t *cov_tab, const uint32_t **row_tab) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint32_t x = root_node[r0 + t];
    cov_tab[t] = cover[x];
    if (row_tab) row_tab[t] = rows + (size_t)slot[x] * W4;
}

// ---- per-program device-plan state ----------------------------------------------------------
struct DPlan {
    const hedl_kb *kb = nullptr;
    uint32_t nn = 0;
    bool lists = false;
    std::vector<uint32_t> lvl_off;             // host: level list offsets
    uint32_t *list = nullptr;                  // canonical nodes by level
    uint8_t *live = nullptr, *isroot = nullptr, *nfull = nullptr, *nproj = nullptr, *pmode = nullptr;
    uint32_t *cover = nullptr, *slot = nullptr, *pslot = nullptr, *bucket = nullptr, *rank_of = nullptr;
    uint32_t *dnode = nullptr, *opfirst = nullptr, *bsum = nullptr, *totals = nullptr, *lhist = nullptr, *lcur = nullptr;
    void *blk = nullptr;                       // pooled block holding the per-node arrays
    size_t blk_bytes = 0;
    uint32_t *bstats = nullptr;                // 5 x nbuckets: count, ops, outs, cov, cursor
    uint32_t *bfirst = nullptr;
    void *bblk = nullptr;
    size_t bcap = 0, bblk_bytes = 0;
    uint32_t *h_stats = nullptr;               // pinned (pooled)
    size_t h_cap = 0;
    ~DPlan() {
        if (blk) pool_give(kb, PR_DPLAN, blk, blk_bytes);
        if (bblk) pool_give(kb, PR_DPLAN, bblk, bblk_bytes);
        if (h_stats) pool_give(kb, PR_DPLAN_HOST, h_stats, h_cap);
    }
    bool alloc(uint32_t n, uint32_t levels) {
        for (int pass = 0; pass < 2; ++pass) {
            Carver c{(char *)blk, 0};
            list = c.take<uint32_t>(n);
            live = c.take<uint8_t>(n); isroot = c.take<uint8_t>(n); nfull = c.take<uint8_t>(n);
            nproj = c.take<uint8_t>(n); pmode = c.take<uint8_t>(n);
            cover = c.take<uint32_t>(n); slot = c.take<uint32_t>(n); pslot = c.take<uint32_t>(n);
            bucket = c.take<uint32_t>(n); rank_of = c.take<uint32_t>(n);
            dnode = c.take<uint32_t>(n); opfirst = c.take<uint32_t>(n);
            bsum = c.take<uint32_t>(nblk(n, 1024) + 1); totals = c.take<uint32_t>(8);
            lhist = c.take<uint32_t>(levels + 2); lcur = c.take<uint32_t>(levels + 2);
            if (pass == 0 && !(blk = pool_alloc(kb, PR_DPLAN, c.off, &blk_bytes))) return false;
        }
        return true;
    }
};

}  // namespace

namespace hedl {

void dplan_free(hedl_program *p) {
    delete (DPlan *)p->dplan;
    p->dplan = nullptr;
}

hedl_status dplan_run(const hedl_kb *kb, hedl_program *p, uint32_t r0, uint32_t r1, uint32_t *out_bits,
                      hedl_counts *counts_dev, cudaStream_t s, uint32_t eflags) {
    Workspace *w = ws_of(p);
    if (w->used && w->last_stream != s && w->done) HEDL_CUDA(kb, cudaStreamWaitEvent(s, w->done, 0));
    PlanCache &pc = w->plan;
    const bool bits = out_bits != nullptr;
    const bool hit = pc.valid && pc.r0 == r0 && pc.r1 == r1 && pc.bits == bits && pc.eflags == eflags &&
                     pc.rows_base == w->rows.p && pc.heavy_base == w->heavy.p && pc.prows_base == w->prows.p;
    hedl_status st;
    if (hit) {
        for (const ChunkPlan &cp : pc.chunks)
            if ((st = launch_chunk(kb, w, cp, r0, out_bits, counts_dev, s))) return st;
    } else {
        if (w->used && w->done) HEDL_CUDA(kb, cudaEventSynchronize(w->done));
        invalidate_plan(pc);
        const double t0 = now_ms();
        const uint32_t nn = p->dev_n_nodes;
        const uint32_t L = p->n_levels;
        if (!p->dplan) {
            DPlan *np = new DPlan();
            np->kb = kb;
            np->nn = nn;
            if (!np->alloc(nn, L)) { delete np; return fail(HEDL_ERR_OOM, "device plan arrays"); }
            p->dplan = np;
        }
        DPlan &D = *(DPlan *)p->dplan;
        if (!D.lists) {                              // canonical level lists (once per program)
            uint32_t *hist = D.lhist, *cur = D.lcur;
            HEDL_CUDA(kb, cudaMemsetAsync(hist, 0, (L + 1) * 4, s));
            if (nn) k_dp_level_hist<<<std::min<uint32_t>(nblk(nn, 1024), 1184), 1024, (L + 1) * 4, s>>>(p->d_nodes, nn, hist, L + 1);
            std::vector<uint32_t> h(L + 1);
            HEDL_CUDA(kb, cudaMemcpyAsync(h.data(), hist, (L + 1) * 4, cudaMemcpyDeviceToHost, s));
            HEDL_CUDA(kb, cudaStreamSynchronize(s));
            D.lvl_off.assign(L + 2, 0);
            for (uint32_t l = 0; l <= L; ++l) D.lvl_off[l + 1] = D.lvl_off[l] + h[l];
            HEDL_CUDA(kb, cudaMemcpyAsync(cur, D.lvl_off.data(), (L + 1) * 4, cudaMemcpyHostToDevice, s));
            if (nn) k_dp_level_scatter<<<nblk(nn, 1024), 1024, 2 * (L + 1) * 4, s>>>(p->d_nodes, nn, cur, D.list, L + 1);
            HEDL_CUDA(kb, cudaStreamSynchronize(s));     // `h` / lvl_off are host memory read by the copies
            D.lists = true;
        }
        auto tsync = [&](const char *what) {          // phase timing (HEDL_TIMING=1 only)
            if (!timing_enabled()) return;
            cudaStreamSynchronize(s);
            timing_note(what, now_ms() - t0);
        };
        tsync("device plan: lists");
        const bool all = r0 == 0 && r1 == p->dev_n_roots;
        // live nodes, roots, demands
        k_dp_init<<<nblk(std::max(nn, 1u), 256), 256, 0, s>>>(p->d_nodes, nn, all, D.live, D.isroot, D.nfull, D.nproj);
        k_dp_roots<<<nblk(r1 - r0, 256), 256, 0, s>>>(p->d_root_node, r0, r1, bits, D.live, D.isroot, D.nfull);
        if (!all)
            for (uint32_t l = L; l-- > 1;) {
                const uint32_t m = D.lvl_off[l + 1] - D.lvl_off[l];
                if (m) k_dp_mark_down<<<nblk(m, 256), 256, 0, s>>>(D.list + D.lvl_off[l], m, p->d_nodes, p->d_ops, D.live);
            }
        for (uint32_t l = L; l-- > 0;) {
            const uint32_t m = D.lvl_off[l + 1] - D.lvl_off[l];
            if (m) k_dp_demand<<<nblk(m, 256), 256, 0, s>>>(D.list + D.lvl_off[l], m, p->d_nodes, p->d_ops, D.live,
                                                             D.nfull, D.nproj, D.pmode);
        }
        tsync("device plan: live+demands");
        scan(s, D.isroot, nn, D.cover, D.bsum, D.totals + 0);
        scan(s, D.nfull, nn, D.slot, D.bsum, D.totals + 1);
        scan(s, D.nproj, nn, D.pslot, D.bsum, D.totals + 2);
        tsync("device plan: scans");
        // groups
        uint32_t dirs = std::max<uint32_t>({1u, 2 * kb->R, kb->D, kb->S});
        const uint64_t nbk = (uint64_t)std::max<uint32_t>(L, 1) * kKinds * dirs * kSub;
        if (nbk > kMaxBuckets) return fail(HEDL_ERR_UNSUPPORTED, "device plan: too many launch groups");
        const BucketGeom g{dirs, (uint32_t)nbk};
        if (D.bcap < nbk) {
            if (D.bblk) pool_give(kb, PR_DPLAN, D.bblk, D.bblk_bytes);
            D.bblk = pool_alloc(kb, PR_DPLAN, nbk * 6 * 4 + 256, &D.bblk_bytes);
            if (!D.bblk) { D.bcap = 0; return fail(HEDL_ERR_OOM, "device plan buckets"); }
            D.bstats = (uint32_t *)D.bblk;
            D.bfirst = D.bstats + nbk * 5;
            D.bcap = nbk;
        }
        const size_t hbytes = nbk * 4 * 4 + 32;
        if (D.h_cap < hbytes) {
            if (D.h_stats) pool_give(kb, PR_DPLAN_HOST, D.h_stats, D.h_cap);
            D.h_stats = nullptr;
            size_t got = 0;
            if (void *q = pool_take(kb, PR_DPLAN_HOST, hbytes, &got)) {
                D.h_stats = (uint32_t *)q;
            } else if (cudaMallocHost((void **)&D.h_stats, hbytes) == cudaSuccess) {
                got = hbytes;
            } else {
                cudaGetLastError();
                D.h_stats = nullptr;
                D.h_cap = 0;
                return fail(HEDL_ERR_OOM, "pinned");
            }
            D.h_cap = got;
        }
        uint32_t *bc = D.bstats, *bo = bc + nbk, *bu = bo + nbk, *bv = bu + nbk, *bcur = bv + nbk;
        HEDL_CUDA(kb, cudaMemsetAsync(D.bstats, 0, nbk * 5 * 4, s));
        if (nn) k_dp_bucket<<<nblk(nn, 256), 256, 0, s>>>(p->d_nodes, nn, D.live, D.pmode, D.nfull, D.nproj, D.isroot, g,
                                                         D.bucket, bc, bo, bu, bv);
        HEDL_CUDA(kb, cudaMemcpyAsync(D.h_stats, D.bstats, nbk * 4 * 4, cudaMemcpyDeviceToHost, s));
        HEDL_CUDA(kb, cudaMemcpyAsync(D.h_stats + nbk * 4, D.totals, 16, cudaMemcpyDeviceToHost, s));
        HEDL_CUDA(kb, cudaStreamSynchronize(s));
        const double t1 = now_ms();
        const uint32_t *hc = D.h_stats, *ho = hc + nbk, *hu = ho + nbk, *hv = hu + nbk, *tot = hv + nbk;
        const uint32_t ncov = tot[0], nrows = tot[1], nprows = tot[2];
        // launch records (ascending bucket = ascending level), descriptor positions per type
        const size_t row_bytes = (size_t)kb->W4 * 4;
        if (!p->ws_limit) {
            size_t fr = 0, tt = 0;
            cudaMemGetInfo(&fr, &tt);
            p->ws_limit = std::max<uint64_t>(1ull << 28, std::min<uint64_t>(fr / 2, 48ull << 30));
        }
        if ((uint64_t)nrows * row_bytes > p->ws_limit)
            return HEDL_ERR_UNSUPPORTED;                 // needs chunking: the host planner's job
        const bool use_slice = !(eflags & HEDL_EVAL_PER_NODE) && slice_enabled(kb);
        const bool force = eflags & HEDL_EVAL_FORCE_SLICE;
        // packable restriction nodes per (level, dir), all demands: the host planner's pack decision
        std::vector<uint32_t> packable((size_t)std::max<uint32_t>(L, 1) * dirs, 0);
        auto bidx = [&](uint32_t l, uint32_t kc, uint32_t dir, uint32_t cls, uint32_t sub) {
            return (((size_t)l * kKinds + kc) * dirs + dir) * kSub + cls * 2 + sub;
        };
        for (uint32_t l = 0; l < L; ++l)
            for (uint32_t d = 0; d < dirs; ++d)
                for (uint32_t c = 0; c < 2; ++c)
                    for (uint32_t sb = 0; sb < 2; ++sb) packable[(size_t)l * dirs + d] += hc[bidx(l, 1, d, c, sb)];
        uint32_t nb = 0, nr = 0, ndr = 0;
        uint64_t n_ops = 0;
        for (uint64_t b = 0; b < nbk; ++b) {
            const uint32_t kc = (uint32_t)((b / kSub / dirs) % kKinds);
            if (kc == 0) { nb += hc[b]; n_ops += ho[b]; }
            else if (kc == 1) nr += hc[b];
            else ndr += hc[b];
        }
        ChunkPlan cp;
        cp.ri = r0;
        cp.rc = r1;
        cp.ncov = ncov;
        cp.nrows = nrows;
        cp.nprows = nprows;
        cp.nn = nb + nr + ndr;
        cp.off_bool = 0;
        cp.off_ops = align_up(nb * sizeof(BoolDesc), 16);
        cp.off_res = align_up(cp.off_ops + n_ops * sizeof(Operand), 16);
        cp.off_dr = align_up(cp.off_res + nr * sizeof(RestrictDesc), 16);
        cp.off_str = align_up(cp.off_dr + ndr * sizeof(DrangeDesc), 16);
        cp.off_cov = cp.off_str;
        const uint32_t nroots = r1 - r0;
        cp.off_rows = align_up(cp.off_cov + nroots * sizeof(uint32_t), 16);
        cp.blob_bytes = align_up(cp.off_rows + (bits ? nroots * sizeof(void *) : 0), 256);
        cp.blob_off = 0;
        std::vector<uint32_t> first(nbk, 0);
        uint32_t cb = 0, cr = 0, cd = 0;
        size_t heavy_need = 16;
        const double W = kb->W, MW = kb->MW;
        for (uint64_t b = 0; b < nbk; ++b) {
            const uint32_t cnt = hc[b];
            if (!cnt) continue;
            const uint32_t sub = b % 2, cls = (uint32_t)((b % kSub) / 2), dir = (uint32_t)((b / kSub) % dirs);
            const uint32_t kc = (uint32_t)((b / kSub / dirs) % kKinds), l = (uint32_t)(b / kSub / dirs / kKinds);
            LaunchRec lr{};
            lr.count = cnt;
            lr.cls = -1;
            if (kc == 0) {
                first[b] = cb;
                lr.kind = NK_AND;
                lr.key = 0;
                lr.proj = sub;
                lr.first_desc = cb;
                lr.bytes = 4.0 * (sub ? MW : W) * ((double)ho[b] + hu[b] + 2.0 * hv[b]);
                cb += cnt;
            } else if (kc == 1) {
                first[b] = nb + cr;
                const hedl_dir &dr = kb->dirs[dir];
                lr.kind = NK_RESTRICT;
                lr.key = (uint16_t)dir;
                lr.first_desc = cr;
                lr.slice = use_slice && cls < 2 && slice_worthwhile(kb, packable[(size_t)l * dirs + dir], force);
                if (lr.slice) {
                    lr.ex = sub;
                    lr.cls = (int8_t)cls;
                } else {
                    heavy_need = std::max(heavy_need, (size_t)cnt * dr.n_heavy * 8);
                    lr.bytes = cnt * (4.0 * (kb->N + 1) + 4.0 * (dr.E - dr.E_heavy)) + 4.0 * W * (cnt + hu[b] + 2.0 * hv[b]);
                    lr.bytes2 = cnt * 4.0 * dr.E_heavy;
                }
                cr += cnt;
            } else {
                first[b] = nb + nr + cd;
                lr.kind = NK_DRANGE;
                lr.key = (uint16_t)dir;
                lr.first_desc = cd;
                lr.bytes = cnt * kb->data_bytes[dir] + 4.0 * W * (hu[b] + 2.0 * hv[b]);
                cd += cnt;
            }
            cp.recs.push_back(lr);
        }
        // buffers (the pointers become final), then the device fill
        if ((st = grow(kb, s, w->rows, (size_t)std::max<uint32_t>(nrows, 1) * row_bytes + 16, false, PR_ROWS))) return st;
        if ((st = grow(kb, s, w->prows, (size_t)std::max<uint32_t>(nprows, 1) * kb->MW4 * 4 + 16, false, PR_PROWS))) return st;
        if ((st = grow(kb, s, w->heavy, heavy_need, true, PR_HEAVY))) return st;
        if ((st = grow(kb, s, w->counts, (size_t)std::max<uint32_t>(ncov, 1) * sizeof(hedl_counts), false, PR_COUNTS))) return st;
        if ((st = reserve_plan(kb, pc, std::max<size_t>(cp.blob_bytes, 256)))) return st;
        std::memcpy(D.h_stats, first.data(), nbk * 4);   // pinned staging (the stats are consumed)
        HEDL_CUDA(kb, cudaMemcpyAsync(D.bfirst, D.h_stats, nbk * 4, cudaMemcpyHostToDevice, s));
        count_io(nbk * 4, 0);
        HEDL_CUDA(kb, cudaMemsetAsync(bcur, 0, nbk * 4, s));
        if (nn) k_dp_scatter<<<nblk(nn, 256), 256, 0, s>>>(nn, D.live, D.bucket, D.bfirst, bcur, D.dnode, D.rank_of);
        if (nb) {
            k_dp_opc<<<nblk(nb, 256), 256, 0, s>>>(D.dnode, nb, p->d_nodes, D.opfirst);
            scan(s, D.opfirst, nb, D.opfirst, D.bsum, D.totals + 3);
        }
        char *blob = (char *)pc.dev;
        FillArgs fa;
        fa.nodes = p->d_nodes; fa.ops = p->d_ops; fa.dnode = D.dnode; fa.rank_of = D.rank_of; fa.opfirst = D.opfirst;
        fa.slot = D.slot; fa.pslot = D.pslot; fa.cover = D.cover;
        fa.nfull = D.nfull; fa.nproj = D.nproj; fa.pmode = D.pmode; fa.isroot = D.isroot;
        fa.nb = nb; fa.nr = nr; fa.nd = ndr;
        fa.bd = (BoolDesc *)(blob + cp.off_bool);
        fa.od = (Operand *)(blob + cp.off_ops);
        fa.rd = (RestrictDesc *)(blob + cp.off_res);
        fa.dd = (DrangeDesc *)(blob + cp.off_dr);
        fa.rows = (uint32_t *)w->rows.p;
        fa.prows = (uint32_t *)w->prows.p;
        fa.concepts = kb->concepts; fa.ones = kb->ones; fa.pconcepts = kb->pconcepts; fa.pones = kb->pones;
        fa.W4 = kb->W4;
        fa.MW4 = kb->MW4;
        for (uint32_t d = 0; d < 64; ++d) fa.n_heavy[d] = d < kb->dirs.size() ? kb->dirs[d].n_heavy : 0;
        if (cp.nn) k_dp_fill<<<nblk(cp.nn, 128), 128, 0, s>>>(fa);
        k_dp_root_tables<<<nblk(nroots, 256), 256, 0, s>>>(p->d_root_node, r0, nroots, D.cover, D.slot, fa.rows, kb->W4,
                                                           (uint32_t *)(blob + cp.off_cov),
                                                           bits ? (const uint32_t **)(blob + cp.off_rows) : nullptr);
        for (int q = 0; q < 8; ++q) count_launch();
        HEDL_CUDA(kb, cudaGetLastError());
        pc.r0 = r0; pc.r1 = r1; pc.bits = bits; pc.eflags = eflags;
        pc.rows_base = w->rows.p;
        pc.heavy_base = w->heavy.p;
        pc.prows_base = w->prows.p;
        pc.chunks.assign(1, std::move(cp));
        timing_note("device plan: groups", t1 - t0);
        if ((st = launch_chunk(kb, w, pc.chunks[0], r0, out_bits, counts_dev, s))) { invalidate_plan(pc); return st; }
        pc.valid = true;
        timing_note("device plan: total", now_ms() - t0);
    }
    if (!w->done) HEDL_CUDA(kb, cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming));
    HEDL_CUDA(kb, cudaEventRecord(w->done, s));
    w->last_stream = s;
    w->used = true;
    return HEDL_OK;
}

}  // namespace hedl

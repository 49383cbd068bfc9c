// Device planner: the evaluation plan of a device-compiled program built
// on the GPU ("each GPU generates its evaluation plans
// ... with minimal to no CPU intervention").
//
// The same plan as the host planner (exec.cu, fill_chunk) for a single chunk: live
// nodes, one count slot per distinct root node, row demands (full rows only for nodes
// another node reads in full, example-projected rows for roots and their operands, U rows
// for the fillers of example-row packs: booleans and ranges evaluated over U, restrictions
// emitting U rows from their full pack), launch groups by (level, kind, direction,
// lane-pack class, demand) plus one group per U direction, descriptors with final device
// addresses.  Every per-node step is a kernel; the host reads back one small table
// (per-group counts, a few KB) to size the buffers and issue the launches.  Boolean
// fillers are not fused into packs here (HEDL_EVAL_NO_FUSE behaviour).
#include <algorithm>

#include "exec.h"
#include "scan.cuh"
#include "slice.h"

using namespace hedl;

namespace {

constexpr uint32_t FULLM = 0xffffffffu;
constexpr uint8_t NK_DEAD_D = 0xff;
constexpr uint32_t kKinds = 4;          // AND/OR, RESTRICT, DRANGE, STRING
constexpr uint32_t kSub = 9;            // class (3) x demand (restriction: full / EX over full rows / EX over U)
constexpr uint32_t kUDirs = 4;          // U directions the device planner handles (kMaxUDirs)
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

// U-capability, bottom up (one level per launch): a node can be evaluated over U_d (DESIGN.md
// "U rows"): restrictions in full lane packs (epilogue), ranges (at the U members), booleans
// whose node operands all can
__global__ void k_dp_ucap(const uint32_t *__restrict__ list, uint32_t m, const CNode *__restrict__ nodes,
                          const uint32_t *__restrict__ ops, uint8_t *ucap, bool u_restr) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t i = list[t];
    const CNode n = nodes[i];
    bool c = false;
    if (n.kind == NK_RESTRICT) c = u_restr && d_slice_class(n.n, n.sat) < 2;
    else if (n.kind == NK_DRANGE) c = u_restr;
    else if (n.kind == NK_AND || n.kind == NK_OR) {
        c = true;
        for (uint32_t q = 0; c && q < n.op_count; ++q) {
            const uint32_t o = ops[n.op_begin + q];
            if (d_isnode(o) && !ucap[o >> 3]) c = false;
        }
    }
    ucap[i] = c;
}

// demands, consumers first (one level per launch, top down; within a level nodes are
// independent, concurrent stores of 1 to a shared operand flag are benign, U demands are
// atomic ORs).  The host planner's rules (exec.cu fill_chunk).
__global__ void k_dp_demand(const uint32_t *__restrict__ list, uint32_t m, const CNode *__restrict__ nodes,
                            const uint32_t *__restrict__ ops, const uint8_t *__restrict__ live,
                            const uint8_t *__restrict__ isroot, const uint8_t *__restrict__ ucap, uint8_t *nfull,
                            uint8_t *nproj, uint8_t *pmode, unsigned long long *needu, unsigned long long *uout,
                            bool use_u) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t i = list[t];
    if (!live[i]) return;
    const CNode n = nodes[i];
    const bool isbool = n.kind == NK_AND || n.kind == NK_OR;
    const unsigned long long nu = needu[i];
    unsigned long long uo = 0;
    if (nu) {
        if (ucap[i]) uo = nu;
        else nfull[i] = 1;                          // the EX packs read its full row
    }
    uout[i] = uo;
    const bool pm = isbool && !nfull[i] && (nproj[i] || isroot[i]);
    pmode[i] = pm;
    const bool ex = use_u && n.kind == NK_RESTRICT && !nfull[i] && !uo && d_slice_class(n.n, n.sat) < 2;
    for (uint32_t q = 0; q < n.op_count; ++q) {
        const uint32_t o = ops[n.op_begin + q];
        if (!d_isnode(o)) continue;
        const uint32_t j = o >> 3;
        if (ex) {
            atomicOr(needu + j, 1ull << (n.dir & 63));
        } else if (!isbool) {
            nfull[j] = 1;
        } else {
            if (nfull[i]) nfull[j] = 1;
            if (pm) nproj[j] = 1;
            if (uo) atomicOr(needu + j, uo);
        }
    }
}

// U-row counts per node, restrictions' rows first (they are atomicOr targets, zeroed per chunk)
__global__ void k_dp_ucount(const CNode *__restrict__ nodes, uint32_t nn, const uint8_t *__restrict__ live,
                            const unsigned long long *__restrict__ uout, uint32_t *cnt_r, uint32_t *cnt_o) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    const uint32_t c = live[i] ? (uint32_t)__popcll(uout[i]) : 0u;
    const bool r = nodes[i].kind == NK_RESTRICT;
    cnt_r[i] = r ? c : 0u;
    cnt_o[i] = r ? 0u : c;
}
__global__ void k_dp_ubase(const CNode *__restrict__ nodes, uint32_t nn, const uint32_t *__restrict__ total_r,
                           const uint32_t *__restrict__ off_r, uint32_t *off_o) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    off_o[i] = nodes[i].kind == NK_RESTRICT ? off_r[i] : *total_r + off_o[i];
}

struct BucketGeom {
    uint32_t dirs, nbuckets;
};

// a restriction evaluated only at the example rows reads its filler over U (the filler is an
// atom / TOP or has a U row of the restriction's direction), else the filler's full row
__device__ __forceinline__ bool d_ex_ucomp(const CNode &n, const uint32_t *__restrict__ ops,
                                           const unsigned long long *__restrict__ uout, bool use_u) {
    const uint32_t c = ops[n.op_begin];
    return use_u && (!d_isnode(c) || ((uout[c >> 3] >> (n.dir & 63)) & 1ull));
}

// the node's main launch group (FULLM: none -- a boolean / range needed only over U)
__device__ __forceinline__ uint32_t d_bucket(const CNode &n, bool pmode, bool nfull, bool nproj, bool root,
                                             unsigned long long uo, const uint32_t *__restrict__ ops,
                                             const unsigned long long *__restrict__ uout, bool use_u,
                                             const BucketGeom &g, uint32_t *cls_out) {
    const uint32_t kc = (n.kind == NK_AND || n.kind == NK_OR) ? 0u : n.kind == NK_RESTRICT ? 1u : n.kind == NK_DRANGE ? 2u : 3u;
    uint32_t cls = 0, sub = 0;
    if (kc == 0) {
        if (!nfull && !pmode) return FULLM;
        sub = pmode;
    } else if (kc == 1) {
        cls = d_slice_class(n.n, n.sat);
        if (cls < 2 && !nfull && !uo) sub = d_ex_ucomp(n, ops, uout, use_u) ? 2u : 1u;
    } else if (kc == 2) {
        if (uo && !nfull && !nproj && !root) return FULLM;
    }
    const uint32_t dir = kc == 0 ? 0u : n.dir;
    *cls_out = cls;
    return ((n.level * kKinds + kc) * g.dirs + dir) * kSub + cls * 3 + sub;
}

// per bucket: count, operands (boolean), rows written, coverage slots
__global__ void k_dp_bucket(const CNode *__restrict__ nodes, const uint32_t *__restrict__ opv, uint32_t nn,
                            const uint8_t *__restrict__ live, const uint8_t *__restrict__ pmode,
                            const uint8_t *__restrict__ nfull, const uint8_t *__restrict__ nproj,
                            const uint8_t *__restrict__ isroot, const unsigned long long *__restrict__ uout, bool use_u,
                            BucketGeom g, uint32_t *bucket, uint32_t *b_count, uint32_t *b_ops, uint32_t *b_outs,
                            uint32_t *b_cov, uint32_t *b_u) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    uint32_t b = FULLM, ops = 0, outs = 0, cov = 0, hu = 0;
    if (i < nn && live[i]) {
        const CNode n = nodes[i];
        uint32_t cls;
        b = d_bucket(n, pmode[i], nfull[i], nproj[i], isroot[i], uout[i], opv, uout, use_u, g, &cls);
        bucket[i] = b;
        if (b != FULLM) {
            const bool isbool = n.kind == NK_AND || n.kind == NK_OR;
            ops = isbool ? n.op_count : 0;
            outs = (isbool && pmode[i]) ? nproj[i] : nfull[i];
            cov = isroot[i];
            hu = n.kind == NK_RESTRICT && uout[i] != 0;
        }
    }
    // warp aggregation by bucket: one atomic per distinct bucket per warp
    const uint32_t peers = __match_any_sync(FULLM, b);
    const uint32_t leader = __ffs(peers) - 1;
    uint32_t s_ops = 0, s_outs = 0, s_cov = 0, s_u = 0;
    for (uint32_t l = 0; l < 32; ++l) {
        const uint32_t a = __shfl_sync(FULLM, ops, l), o = __shfl_sync(FULLM, outs, l), c = __shfl_sync(FULLM, cov, l);
        const uint32_t h = __shfl_sync(FULLM, hu, l);
        if (peers & (1u << l)) { s_ops += a; s_outs += o; s_cov += c; s_u += h; }
    }
    if (b != FULLM && lane == leader) {
        atomicAdd(b_count + b, (uint32_t)__popc(peers));
        if (s_ops) atomicAdd(b_ops + b, s_ops);
        if (s_outs) atomicAdd(b_outs + b, s_outs);
        if (s_cov) atomicAdd(b_cov + b, s_cov);
        if (s_u) atomicAdd(b_u + b, s_u);
    }
}

// U entries: one (node, direction) pair per U row a boolean / range computes; U bucket =
// (level, booleans | the range's data property, direction); counted, then scattered
__device__ __forceinline__ uint32_t d_ubucket(uint32_t level, bool drange, uint32_t prop, uint32_t nprop, uint32_t d) {
    return (level * (1 + nprop) + (drange ? 1 + prop : 0u)) * kUDirs + d;
}
__global__ void k_dp_ucnt(const CNode *__restrict__ nodes, uint32_t nn, const uint8_t *__restrict__ live,
                          const unsigned long long *__restrict__ uout, uint32_t nprop, uint32_t *u_count, uint32_t *u_ops) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn || !live[i]) return;
    const CNode n = nodes[i];
    if (n.kind == NK_RESTRICT || !uout[i]) return;
    const bool dr = n.kind == NK_DRANGE;
    for (unsigned long long m = uout[i]; m; m &= m - 1) {
        const uint32_t ub = d_ubucket(n.level, dr, n.dir, nprop, (uint32_t)__ffsll(m) - 1);
        atomicAdd(u_count + ub, 1u);
        if (!dr) atomicAdd(u_ops + ub, n.op_count);
    }
}
__global__ void k_dp_uscatter(const CNode *__restrict__ nodes, uint32_t nn, const uint8_t *__restrict__ live,
                              const unsigned long long *__restrict__ uout, uint32_t nprop, const uint32_t *__restrict__ u_first,
                              uint32_t *u_cur, uint32_t *udnode, uint8_t *udir) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn || !live[i]) return;
    const CNode n = nodes[i];
    if (n.kind == NK_RESTRICT || !uout[i]) return;
    const bool dr = n.kind == NK_DRANGE;
    for (unsigned long long m = uout[i]; m; m &= m - 1) {
        const uint32_t d = (uint32_t)__ffsll(m) - 1, ub = d_ubucket(n.level, dr, n.dir, nprop, d);
        const uint32_t pos = u_first[ub] + atomicAdd(u_cur + ub, 1u);
        udnode[pos] = i;
        udir[pos] = (uint8_t)d;
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

// operand counts of every boolean descriptor: main ones (dnode), then U entries (udnode)
__global__ void k_dp_opc(const uint32_t *__restrict__ dnode, uint32_t nbm, const uint32_t *__restrict__ udnode,
                         uint32_t nbu, const CNode *__restrict__ nodes, uint32_t *opc) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nbm) opc[t] = nodes[dnode[t]].op_count;
    else if (t < nbm + nbu) opc[t] = nodes[udnode[t - nbm]].op_count;
}

struct FillArgs {
    const CNode *nodes;
    const uint32_t *ops;
    const uint32_t *dnode, *rank_of, *opfirst, *slot, *pslot, *cover;
    const uint8_t *nfull, *nproj, *pmode, *isroot;
    uint32_t nb, nr, nd;                  // main descriptor counts per type (bool, restrict, range)
    // U rows: per node the directions and first slot; U entries (bool / range over U_d)
    const unsigned long long *uout;
    const uint32_t *ubase, *udnode;
    const uint8_t *udir;
    uint32_t nbu, ndu, ustride;
    bool use_u;
    uint32_t *urows;
    const uint32_t *uconcepts[kUDirs], *uones[kUDirs];
    uint32_t uw4[kUDirs];
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
__device__ __forceinline__ uint32_t *d_urow(const FillArgs &a, uint32_t node, uint32_t d) {
    return a.urows + (size_t)(a.ubase[node] + __popcll(a.uout[node] & ((1ull << d) - 1ull))) * a.ustride;
}
__device__ __forceinline__ const uint32_t *d_uptr_of(const FillArgs &a, uint32_t r, uint32_t d) {
    const uint32_t t = (r >> 1) & 3u, id = r >> 3;
    if (t == RT_NODE) return d_urow(a, id, d);
    if (t == RT_ATOM) return a.uconcepts[d] + (size_t)id * a.uw4[d];
    return a.uones[d];
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
        const unsigned long long uo = a.uout[k];
        const bool ex = a.use_u && !a.nfull[k] && !uo && d_slice_class(n.n, n.sat) < 2;
        // an example-row pack over U reads the filler's U row of this direction
        d.child = (ex && d_ex_ucomp(n, a.ops, a.uout, a.use_u)) ? d_uptr_of(a, c, n.dir) : d_ptr_of(a, c);
        d.out = out;
        d.proj = proj;
        d.cmask = (c & 1u) ? 0xffffffffu : 0u;
        d.pred = n.pred;
        d.n = n.n;
        d.sat = n.sat;
        d.cover = cover;
        d.heavy_slot = a.rank_of[k] * a.n_heavy[n.dir & 63];
        d.op_first = d.op_n = 0;
        d.uout = uo ? d_urow(a, k, (uint32_t)__ffsll(uo) - 1) : nullptr;   // U rows from the pack epilogue
        d.udirs = (uint32_t)uo;
        d.pad_ = 0;
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

// U entries: booleans evaluated over U_d (operands' U rows), ranges at the members of U_d
__global__ void k_dp_fill_u(FillArgs a) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.nbu + a.ndu) return;
    const uint32_t k = a.udnode[t], dd = a.udir[t];
    const CNode n = a.nodes[k];
    if (t < a.nbu) {
        BoolDesc d;
        d.out = d_urow(a, k, dd);
        d.proj = nullptr;
        d.op_first = a.opfirst[a.nb + t];
        d.op_count = n.op_count;
        d.is_or = n.kind == NK_OR;
        d.cover = -1;
        for (uint32_t q = 0; q < n.op_count; ++q) {
            const uint32_t o = a.ops[n.op_begin + q];
            a.od[d.op_first + q] = Operand{d_uptr_of(a, o, dd), (o & 1u) ? 0xffffffffu : 0u, 0};
        }
        a.bd[a.nb + t] = d;
    } else {
        DrangeDesc d;
        d.out = d_urow(a, k, dd);
        d.proj = nullptr;
        d.lo = n.lo;
        d.hi = n.hi;
        d.cover = -1;
        d.prop = n.dir;
        a.dd[a.nd + (t - a.nbu)] = d;
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
    uint8_t *live = nullptr, *isroot = nullptr, *nfull = nullptr, *nproj = nullptr, *pmode = nullptr, *ucap = nullptr;
    uint32_t *cover = nullptr, *slot = nullptr, *pslot = nullptr, *bucket = nullptr, *rank_of = nullptr;
    uint32_t *dnode = nullptr, *opfirst = nullptr, *bsum = nullptr, *totals = nullptr, *lhist = nullptr, *lcur = nullptr;
    unsigned long long *needu = nullptr, *uout = nullptr;
    uint32_t *ucnt_r = nullptr, *ucnt_o = nullptr, *ubase = nullptr, *udnode = nullptr;
    uint8_t *udir = nullptr;
    void *blk = nullptr;                       // pooled block holding the per-node arrays
    size_t blk_bytes = 0;
    uint32_t *bstats = nullptr;                // 6 x nbuckets: count, ops, outs, cov, U emitters, cursor
    uint32_t *bfirst = nullptr;
    void *bblk = nullptr;
    size_t bcap = 0, bblk_bytes = 0;
    uint32_t *h_stats = nullptr;               // pinned (pooled)
    size_t h_cap = 0;
    size_t opfirst_cap = 0;
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
            nproj = c.take<uint8_t>(n); pmode = c.take<uint8_t>(n); ucap = c.take<uint8_t>(n);
            needu = c.take<unsigned long long>(n); uout = c.take<unsigned long long>(n);
            ucnt_r = c.take<uint32_t>(n); ucnt_o = c.take<uint32_t>(n); ubase = c.take<uint32_t>(n);
            udnode = c.take<uint32_t>((size_t)n * kUDirs); udir = c.take<uint8_t>((size_t)n * kUDirs);
            opfirst_cap = (size_t)n * (kUDirs + 1);
            cover = c.take<uint32_t>(n); slot = c.take<uint32_t>(n); pslot = c.take<uint32_t>(n);
            bucket = c.take<uint32_t>(n); rank_of = c.take<uint32_t>(n);
            dnode = c.take<uint32_t>(n); opfirst = c.take<uint32_t>((size_t)n * (kUDirs + 1));
            bsum = c.take<uint32_t>(nblk((uint64_t)n * (kUDirs + 1), 1024) + 1); totals = c.take<uint32_t>(8);
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
                     pc.rows_base == w->rows.p && pc.heavy_base == w->heavy.p && pc.prows_base == w->prows.p &&
                     pc.urows_base == w->urows.p;
    hedl_status st;
    if (hit) {
        if ((st = replay_plan(kb, w, r0, out_bits, counts_dev, s))) return st;
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
        const bool use_slice = !(eflags & HEDL_EVAL_PER_NODE) && slice_enabled(kb);
        const bool force = eflags & HEDL_EVAL_FORCE_SLICE;
        // U rows: fillers of example-row packs evaluated over U_d
        const bool use_u = use_slice && kb->M > 0 && kb->dirs.size() <= kUDirs;
        const bool u_restr = use_u && !(eflags & HEDL_EVAL_NO_RESTRICT_U);
        const bool all = r0 == 0 && r1 == p->dev_n_roots;
        // live nodes, roots, U capability (bottom up), demands (top down)
        HEDL_CUDA(kb, cudaMemsetAsync(D.totals, 0, 8 * 4, s));   // (all 8 are read back below)
        k_dp_init<<<nblk(std::max(nn, 1u), 256), 256, 0, s>>>(p->d_nodes, nn, all, D.live, D.isroot, D.nfull, D.nproj);
        if (nn) {
            HEDL_CUDA(kb, cudaMemsetAsync(D.needu, 0, (size_t)nn * 8, s));
            HEDL_CUDA(kb, cudaMemsetAsync(D.uout, 0, (size_t)nn * 8, s));
            HEDL_CUDA(kb, cudaMemsetAsync(D.ucap, 0, nn, s));
        }
        k_dp_roots<<<nblk(r1 - r0, 256), 256, 0, s>>>(p->d_root_node, r0, r1, bits, D.live, D.isroot, D.nfull);
        if (!all)
            for (uint32_t l = L; l-- > 1;) {
                const uint32_t m = D.lvl_off[l + 1] - D.lvl_off[l];
                if (m) k_dp_mark_down<<<nblk(m, 256), 256, 0, s>>>(D.list + D.lvl_off[l], m, p->d_nodes, p->d_ops, D.live);
            }
        if (use_u)
            for (uint32_t l = 0; l < L; ++l) {
                const uint32_t m = D.lvl_off[l + 1] - D.lvl_off[l];
                if (m) k_dp_ucap<<<nblk(m, 256), 256, 0, s>>>(D.list + D.lvl_off[l], m, p->d_nodes, p->d_ops, D.ucap, u_restr);
            }
        for (uint32_t l = L; l-- > 0;) {
            const uint32_t m = D.lvl_off[l + 1] - D.lvl_off[l];
            if (m) k_dp_demand<<<nblk(m, 256), 256, 0, s>>>(D.list + D.lvl_off[l], m, p->d_nodes, p->d_ops, D.live, D.isroot,
                                                             D.ucap, D.nfull, D.nproj, D.pmode, D.needu, D.uout, use_u);
        }
        tsync("device plan: live+demands");
        scan(s, D.isroot, nn, D.cover, D.bsum, D.totals + 0);
        scan(s, D.nfull, nn, D.slot, D.bsum, D.totals + 1);
        scan(s, D.nproj, nn, D.pslot, D.bsum, D.totals + 2);
        if (use_u && nn) {                           // U-row slots, restrictions' first
            k_dp_ucount<<<nblk(nn, 256), 256, 0, s>>>(p->d_nodes, nn, D.live, D.uout, D.ucnt_r, D.ucnt_o);
            scan(s, D.ucnt_r, nn, D.ucnt_r, D.bsum, D.totals + 4);
            scan(s, D.ucnt_o, nn, D.ubase, D.bsum, D.totals + 5);
            k_dp_ubase<<<nblk(nn, 256), 256, 0, s>>>(p->d_nodes, nn, D.totals + 4, D.ucnt_r, D.ubase);
        } else {
            HEDL_CUDA(kb, cudaMemsetAsync(D.totals + 4, 0, 8, s));
        }
        tsync("device plan: scans");
        // groups: main buckets + U buckets
        uint32_t dirs = std::max<uint32_t>({1u, 2 * kb->R, kb->D, kb->S});
        const uint64_t nbk = (uint64_t)std::max<uint32_t>(L, 1) * kKinds * dirs * kSub;
        const uint32_t nprop = kb->D;
        const uint64_t nub = (uint64_t)std::max<uint32_t>(L, 1) * (1 + nprop) * kUDirs;
        if (nbk > kMaxBuckets) return fail(HEDL_ERR_UNSUPPORTED, "device plan: too many launch groups");
        const BucketGeom g{dirs, (uint32_t)nbk};
        const size_t nstat = nbk * 6 + nub * 4;      // main: 5 stats + cursor; U: count, ops, first, cursor
        if (D.bcap < nstat) {
            if (D.bblk) pool_give(kb, PR_DPLAN, D.bblk, D.bblk_bytes);
            D.bblk = pool_alloc(kb, PR_DPLAN, (nstat + nbk) * 4 + 256, &D.bblk_bytes);
            if (!D.bblk) { D.bcap = 0; return fail(HEDL_ERR_OOM, "device plan buckets"); }
            D.bstats = (uint32_t *)D.bblk;
            D.bfirst = D.bstats + nstat;
            D.bcap = nstat;
        }
        const size_t hbytes = (nbk * 5 + nub * 2) * 4 + 64;
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
        uint32_t *bc = D.bstats, *bo = bc + nbk, *bu = bo + nbk, *bv = bu + nbk, *bh = bv + nbk, *bcur = bh + nbk;
        uint32_t *uc = bcur + nbk, *uo = uc + nub, *ufirst = uo + nub, *ucur = ufirst + nub;
        HEDL_CUDA(kb, cudaMemsetAsync(D.bstats, 0, nstat * 4, s));
        if (nn) k_dp_bucket<<<nblk(nn, 256), 256, 0, s>>>(p->d_nodes, p->d_ops, nn, D.live, D.pmode, D.nfull, D.nproj,
                                                         D.isroot, D.uout, use_u, g, D.bucket, bc, bo, bu, bv, bh);
        if (nn && use_u) k_dp_ucnt<<<nblk(nn, 256), 256, 0, s>>>(p->d_nodes, nn, D.live, D.uout, nprop, uc, uo);
        uint32_t *hs = D.h_stats;
        HEDL_CUDA(kb, cudaMemcpyAsync(hs, D.bstats, nbk * 5 * 4, cudaMemcpyDeviceToHost, s));
        HEDL_CUDA(kb, cudaMemcpyAsync(hs + nbk * 5, uc, nub * 2 * 4, cudaMemcpyDeviceToHost, s));
        HEDL_CUDA(kb, cudaMemcpyAsync(hs + nbk * 5 + nub * 2, D.totals, 32, cudaMemcpyDeviceToHost, s));
        HEDL_CUDA(kb, cudaStreamSynchronize(s));
        const double t1 = now_ms();
        const uint32_t *hc = hs, *ho = hc + nbk, *hu = ho + nbk, *hv = hu + nbk, *hh = hv + nbk;
        const uint32_t *huc = hs + nbk * 5, *huo = huc + nub, *tot = huc + 2 * nub;
        const uint32_t ncov = tot[0], nrows = tot[1], nprows = tot[2], nur_r = tot[4], nur_o = tot[5];
        // launch records, descriptor positions per type
        const size_t row_bytes = (size_t)kb->W4 * 4;
        if (!p->ws_limit) {
            size_t fr = 0, tt = 0;
            cudaMemGetInfo(&fr, &tt);
            p->ws_limit = std::max<uint64_t>(1ull << 28, std::min<uint64_t>(fr / 2, 48ull << 30));
        }
        if ((uint64_t)nrows * row_bytes > p->ws_limit)
            return HEDL_ERR_UNSUPPORTED;                 // needs chunking: the host planner's job
        auto bidx = [&](uint32_t l, uint32_t kc, uint32_t dir, uint32_t cls, uint32_t sub) {
            return (((size_t)l * kKinds + kc) * dirs + dir) * kSub + cls * 3 + sub;
        };
        auto ubidx = [&](uint32_t l, uint32_t grp, uint32_t d) { return ((size_t)l * (1 + nprop) + grp) * kUDirs + d; };
        uint32_t nb = 0, nr = 0, ndr = 0, nbu = 0, ndu = 0;
        uint64_t n_ops = 0;
        for (uint64_t b = 0; b < nbk; ++b) {
            const uint32_t kc = (uint32_t)((b / kSub / dirs) % kKinds);
            if (kc == 0) { nb += hc[b]; n_ops += ho[b]; }
            else if (kc == 1) nr += hc[b];
            else ndr += hc[b];
        }
        std::vector<uint32_t> ufirst_h(nub, 0);
        for (uint32_t dr = 0; dr < 2; ++dr)              // U booleans first, then U ranges
            for (uint32_t l = 0; l < std::max<uint32_t>(L, 1); ++l)
                for (uint32_t grp = dr ? 1 : 0; grp < (dr ? 1 + nprop : 1); ++grp)
                    for (uint32_t d = 0; d < kUDirs; ++d) {
                        const size_t ub = ubidx(l, grp, d);
                        ufirst_h[ub] = nbu + ndu;
                        if (dr == 0) { nbu += huc[ub]; n_ops += huo[ub]; }
                        else ndu += huc[ub];
                    }
        ChunkPlan cp;
        cp.ri = r0;
        cp.rc = r1;
        cp.ncov = ncov;
        cp.nrows = nrows;
        cp.nprows = nprows;
        cp.nurows = nur_r + nur_o;
        cp.nurows_r = nur_r;
        cp.nn = nb + nr + ndr;
        cp.off_bool = 0;
        cp.off_ops = align_up((size_t)(nb + nbu) * sizeof(BoolDesc), 16);
        cp.off_res = align_up(cp.off_ops + n_ops * sizeof(Operand), 16);
        cp.off_dr = align_up(cp.off_res + nr * sizeof(RestrictDesc), 16);
        cp.off_str = align_up(cp.off_dr + (size_t)(ndr + ndu) * sizeof(DrangeDesc), 16);
        cp.off_cov = cp.off_str;
        const uint32_t nroots = r1 - r0;
        cp.off_rows = align_up(cp.off_cov + nroots * sizeof(uint32_t), 16);
        cp.blob_bytes = align_up(cp.off_rows + (bits ? nroots * sizeof(void *) : 0), 256);
        cp.blob_off = 0;
        std::vector<uint32_t> first(nbk, 0);
        uint32_t cb = 0, cr = 0, cd = 0;
        size_t heavy_need = 16;
        const double W = kb->W, MW = kb->MW;
        const uint32_t per_level = kKinds * dirs * kSub;
        for (uint32_t l = 0; l < std::max<uint32_t>(L, 1); ++l) {
            for (uint64_t b = (uint64_t)l * per_level; b < (uint64_t)(l + 1) * per_level; ++b) {
                const uint32_t cnt = hc[b];
                if (!cnt) continue;
                const uint32_t sub = (uint32_t)(b % 3), cls = (uint32_t)((b % kSub) / 3), dir = (uint32_t)((b / kSub) % dirs);
                const uint32_t kc = (uint32_t)((b / kSub / dirs) % kKinds);
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
                    if (sub) {                               // example rows only: always packed
                        lr.slice = true;
                        lr.ex = true;
                        lr.ucomp = sub == 2;
                        lr.cls = (int8_t)cls;
                    } else {
                        // full members of (level, dir): the host planner's pack decision; restrictions
                        // emitting U rows force it (the epilogue is the pack's)
                        uint32_t nf = 0;
                        for (uint32_t c2 = 0; c2 < 2; ++c2) nf += hc[bidx(l, 1, dir, c2, 0)];
                        lr.slice = use_slice && cls < 2 && (slice_worthwhile(kb, nf, force) || hh[b] > 0);
                        if (lr.slice) {
                            lr.cls = (int8_t)cls;
                        } else {
                            heavy_need = std::max(heavy_need, restrict_scratch_bytes(kb, dir, cnt));
                            lr.bytes = cnt * (4.0 * (kb->N + 1) + 4.0 * (dr.E - dr.E_heavy)) + 4.0 * W * (cnt + hu[b] + 2.0 * hv[b]);
                            lr.bytes2 = cnt * 4.0 * dr.E_heavy;
                        }
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
            for (uint32_t grp = 0; grp < 1 + nprop && use_u; ++grp)     // this level's U groups
                for (uint32_t d = 0; d < kUDirs; ++d) {
                    const uint32_t dr = grp > 0;
                    const size_t ub = ubidx(l, grp, d);
                    if (!huc[ub]) continue;
                    LaunchRec lr{};
                    lr.count = huc[ub];
                    lr.cls = -1;
                    lr.usp = (int16_t)d;
                    if (dr == 0) {
                        lr.kind = NK_AND;
                        lr.key = 0;
                        lr.first_desc = nb + ufirst_h[ub];
                        lr.bytes = 4.0 * kb->dirs[d].UW * ((double)huo[ub] + huc[ub]);
                    } else {
                        lr.kind = NK_DRANGE;
                        lr.key = (uint16_t)(grp - 1);        // the data property
                        lr.first_desc = ndr + (ufirst_h[ub] - nbu);
                        lr.bytes = 4.0 * kb->dirs[d].n_u * 3.0 * huc[ub];
                    }
                    cp.recs.push_back(lr);
                }
        }
        // buffers (the pointers become final), then the device fill
        uint32_t uw4max = 0;
        for (const hedl_dir &x : kb->dirs) uw4max = std::max(uw4max, x.UW4);
        if ((st = grow(kb, s, w->rows, (size_t)std::max<uint32_t>(nrows, 1) * row_bytes + 16, false, PR_ROWS))) return st;
        if ((st = grow(kb, s, w->prows, (size_t)std::max<uint32_t>(nprows, 1) * kb->MW4 * 4 + 16, false, PR_PROWS))) return st;
        if ((st = grow(kb, s, w->urows, (size_t)std::max<uint32_t>(cp.nurows, 1) * uw4max * 4 + 16, false, PR_UROWS))) return st;
        if ((st = grow(kb, s, w->heavy, heavy_need, true, PR_HEAVY))) return st;
        if ((st = grow(kb, s, w->counts, (size_t)std::max<uint32_t>(ncov, 1) * sizeof(hedl_counts), false, PR_COUNTS))) return st;
        if ((st = reserve_plan(kb, pc, std::max<size_t>(cp.blob_bytes, 256)))) return st;
        std::memcpy(D.h_stats, first.data(), nbk * 4);   // pinned staging (the stats are consumed)
        std::memcpy(D.h_stats + nbk, ufirst_h.data(), nub * 4);
        HEDL_CUDA(kb, cudaMemcpyAsync(D.bfirst, D.h_stats, nbk * 4, cudaMemcpyHostToDevice, s));
        HEDL_CUDA(kb, cudaMemcpyAsync(ufirst, D.h_stats + nbk, nub * 4, cudaMemcpyHostToDevice, s));
        count_io((nbk + nub) * 4, 0);
        HEDL_CUDA(kb, cudaMemsetAsync(bcur, 0, nbk * 4, s));
        HEDL_CUDA(kb, cudaMemsetAsync(ucur, 0, nub * 4, s));
        if (nn) k_dp_scatter<<<nblk(nn, 256), 256, 0, s>>>(nn, D.live, D.bucket, D.bfirst, bcur, D.dnode, D.rank_of);
        if (nn && (nbu + ndu))
            k_dp_uscatter<<<nblk(nn, 256), 256, 0, s>>>(p->d_nodes, nn, D.live, D.uout, nprop, ufirst, ucur, D.udnode, D.udir);
        if (nb + nbu) {
            k_dp_opc<<<nblk(nb + nbu, 256), 256, 0, s>>>(D.dnode, nb, D.udnode, nbu, p->d_nodes, D.opfirst);
            scan(s, D.opfirst, nb + nbu, D.opfirst, D.bsum, D.totals + 3);
        }
        char *blob = (char *)pc.dev;
        FillArgs fa;
        fa.nodes = p->d_nodes; fa.ops = p->d_ops; fa.dnode = D.dnode; fa.rank_of = D.rank_of; fa.opfirst = D.opfirst;
        fa.slot = D.slot; fa.pslot = D.pslot; fa.cover = D.cover;
        fa.nfull = D.nfull; fa.nproj = D.nproj; fa.pmode = D.pmode; fa.isroot = D.isroot;
        fa.nb = nb; fa.nr = nr; fa.nd = ndr;
        fa.uout = D.uout; fa.ubase = D.ubase; fa.udnode = D.udnode; fa.udir = D.udir;
        fa.nbu = nbu; fa.ndu = ndu; fa.ustride = uw4max; fa.use_u = use_u;
        fa.urows = (uint32_t *)w->urows.p;
        for (uint32_t d = 0; d < kUDirs; ++d) {
            const bool has = d < kb->dirs.size();
            fa.uconcepts[d] = has ? kb->dirs[d].uconcepts : nullptr;
            fa.uones[d] = has ? kb->dirs[d].uones : nullptr;
            fa.uw4[d] = has ? kb->dirs[d].UW4 : 0;
        }
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
        if (nbu + ndu) k_dp_fill_u<<<nblk(nbu + ndu, 128), 128, 0, s>>>(fa);
        k_dp_root_tables<<<nblk(nroots, 256), 256, 0, s>>>(p->d_root_node, r0, nroots, D.cover, D.slot, fa.rows, kb->W4,
                                                           (uint32_t *)(blob + cp.off_cov),
                                                           bits ? (const uint32_t **)(blob + cp.off_rows) : nullptr);
        for (int q = 0; q < 8; ++q) count_launch();
        HEDL_CUDA(kb, cudaGetLastError());
        pc.r0 = r0; pc.r1 = r1; pc.bits = bits; pc.eflags = eflags;
        pc.rows_base = w->rows.p;
        pc.heavy_base = w->heavy.p;
        pc.prows_base = w->prows.p;
        pc.urows_base = w->urows.p;
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

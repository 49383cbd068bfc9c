// hedl_compile_device: hypothesis node arrays already in device memory -> canonical DAG
// program, built on the GPU (the paper's future work, PAPER.md:872:
// "each GPU generates its evaluation plans for its assigned hypotheses with minimal to no
// CPU intervention").
//
// Same canonical form as the host compiler (compile.cpp): complement folded into operand
// references, AND/OR flattened / sorted / deduplicated, hash-consed nodes (CSE across the
// whole batch), topological levels, per-node algorithmic bytes.  Steps (all device work,
// a handful of small D2H reads for grid sizes and the error word):
//   1. input levels by relaxation (children precede parents in the input, so every pass
//      is a parallel sweep; it converges after depth passes), structural checks;
//   2. level lists (histogram + scatter), reachability from the roots, level by level down;
//   3. validation of the reachable nodes (first failing node reported);
//   4. canonicalisation level by level up: one thread per input node builds its canonical
//      node and interns it in a lock-free open-addressing table (materialise, fence, CAS;
//      a thread that loses the race leaves a dead hole, as the host merge does);
//   5. roots: a non-node or complemented root gets a one-operand AND wrapper.
#include <cuda/atomic>

#include <algorithm>

#include "internal.h"

using namespace hedl;

namespace {

constexpr uint32_t kDcMaxOps = 64;       // AND/OR operands after flattening (device limit)
constexpr uint32_t kDcMaxDepth = 512;    // relaxation passes (input depth) before giving up
constexpr uint8_t NK_DEAD_DEV = 0xff;    // same marker as compile.cpp's NK_DEAD

enum DcErr : uint32_t {
    DE_NONE = 0, DE_CHILD_RANGE, DE_CHILD_ORDER, DE_OPCODE, DE_FLAGS, DE_INV_NONROLE, DE_ARITY_LEAF,
    DE_ARITY_NOT, DE_ARITY_ROLE, DE_ATOM_RANGE, DE_ROLE_RANGE, DE_DATA_RANGE, DE_N_BIG, DE_NAN, DE_STRING,
    DE_OPS_LIMIT, DE_OPS_CAP, DE_ROOT_RANGE, DE_DEPTH
};

struct DcErrInfo { hedl_status st; const char *msg; };
const DcErrInfo kDcErr[] = {
    {HEDL_OK, ""},
    {HEDL_ERR_OUT_OF_RANGE, "child id or child range out of range"},
    {HEDL_ERR_BAD_EXPR, "device compile needs children before parents (child id < node id)"},
    {HEDL_ERR_BAD_EXPR, "unknown opcode"},
    {HEDL_ERR_BAD_EXPR, "unknown flag bits"},
    {HEDL_ERR_BAD_EXPR, "inverse flag on a non-role node"},
    {HEDL_ERR_BAD_EXPR, "TOP/BOTTOM/ATOM/DRANGE take no children"},
    {HEDL_ERR_BAD_EXPR, "NOT takes one child"},
    {HEDL_ERR_BAD_EXPR, "role restriction takes one child"},
    {HEDL_ERR_OUT_OF_RANGE, "concept id out of range"},
    {HEDL_ERR_OUT_OF_RANGE, "role id out of range"},
    {HEDL_ERR_OUT_OF_RANGE, "data property id out of range"},
    {HEDL_ERR_BAD_EXPR, "n > 2^32-2"},
    {HEDL_ERR_BAD_EXPR, "NaN bound"},
    {HEDL_ERR_UNSUPPORTED, "string restrictions need hedl_compile_ex (host patterns)"},
    {HEDL_ERR_UNSUPPORTED, "AND/OR with more than 64 operands after flattening (use hedl_compile)"},
    {HEDL_ERR_OOM, "operand table overflow"},
    {HEDL_ERR_OUT_OF_RANGE, "root out of range"},
    {HEDL_ERR_UNSUPPORTED, "input deeper than 512 levels (use hedl_compile)"},
};

struct DcCounters {
    uint32_t n_nodes;
    uint32_t max_level;
    unsigned long long n_ops;
    unsigned long long err;     // (node << 8) | code, minimum wins; ~0 = none
    uint32_t changed;
    uint32_t lvl_max;           // largest level assigned (levels only grow: the last pass's is exact)
};

struct DcKb {                    // what the device compiler needs of the KB
    uint32_t C, R, D, W;
    const double *dir_bytes;     // [2R]
    const double *data_bytes;    // [D]
};

__device__ __forceinline__ void dc_error(DcCounters *c, uint64_t node, uint32_t code) {
    atomicMin(&c->err, (unsigned long long)((node << 8) | code));
}

__device__ __forceinline__ uint32_t d_mkref(uint32_t t, uint32_t id, uint32_t comp) { return (id << 3) | (t << 1) | comp; }

__device__ __forceinline__ uint64_t d_mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h * 0xff51afd7ed558ccdull;
}

__device__ uint64_t d_hash(const CNode &n, const uint32_t *ops) {
    uint64_t h = d_mix(n.kind, n.pred);
    h = d_mix(h, n.dir);
    h = d_mix(h, n.n);
    h = d_mix(h, ((uint64_t)__float_as_uint(n.lo) << 32) | __float_as_uint(n.hi));
    for (uint32_t i = 0; i < n.op_count; ++i) h = d_mix(h, ops[i]);
    return h;
}

__device__ bool d_same(const CNode &a, const uint32_t *aops, const CNode &b, const uint32_t *bops) {
    if (a.kind != b.kind || a.pred != b.pred || a.dir != b.dir || a.n != b.n || a.op_count != b.op_count) return false;
    if (__float_as_uint(a.lo) != __float_as_uint(b.lo) || __float_as_uint(a.hi) != __float_as_uint(b.hi)) return false;
    for (uint32_t i = 0; i < a.op_count; ++i)
        if (aops[i] != bops[i]) return false;
    return true;
}

// ---- 1. levels ----------------------------------------------------------------------
__global__ void k_dc_level(const hedl_node *__restrict__ nodes, uint32_t n, const uint32_t *__restrict__ kids,
                           uint64_t n_kids, uint32_t *lvl, uint8_t *bad, DcCounters *cnt) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    bool changed = false;
    uint32_t lmax = 0;
    if (i < n) {
        const hedl_node nd = nodes[i];
        uint32_t L = 0;
        uint8_t b = 0;
        if ((uint64_t)nd.child_begin + nd.child_count > n_kids) {
            b = DE_CHILD_RANGE;
        } else {
            for (uint32_t k = 0; k < nd.child_count; ++k) {
                const uint32_t c = kids[nd.child_begin + k];
                if (c >= i) { b = c >= n ? DE_CHILD_RANGE : DE_CHILD_ORDER; break; }
                L = max(L, ((volatile uint32_t *)lvl)[c] + 1);
            }
        }
        if (b) { bad[i] = b; L = 0; }
        if (L != lvl[i]) {
            lvl[i] = L;
            changed = true;
        }
        lmax = max(lmax, L);
    }
    if (__any_sync(0xffffffffu, changed) && (threadIdx.x & 31) == 0) cnt->changed = 1;
    lmax = __reduce_max_sync(0xffffffffu, lmax);
    if ((threadIdx.x & 31) == 0 && lmax) atomicMax(&cnt->lvl_max, lmax);
}

// One pass instead of depth + 1 relaxation passes (each a launch and a host round trip): a
// thread computes its node's level exactly by a bounded depth-first walk of its sub-DAG
// (children have smaller indices; hypotheses are small trees).  A walk deeper than kDfsDepth
// or longer than kDfsVisits leaves a lower bound and requests the relaxation passes, which
// converge from there.
constexpr int kDfsDepth = 12;
constexpr uint32_t kDfsVisits = 96;
__global__ void k_dc_level_dfs(const hedl_node *__restrict__ nodes, uint32_t n, const uint32_t *__restrict__ kids,
                               uint64_t n_kids, uint32_t *lvl, uint8_t *bad, DcCounters *cnt) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    bool again = false;
    uint32_t lmax = 0;
    if (i < n) {
        const hedl_node nd = nodes[i];
        uint8_t b = 0;
        if ((uint64_t)nd.child_begin + nd.child_count > n_kids) {
            b = DE_CHILD_RANGE;
        } else {
            for (uint32_t k = 0; k < nd.child_count; ++k) {
                const uint32_t c = kids[nd.child_begin + k];
                if (c >= i) { b = c >= n ? DE_CHILD_RANGE : DE_CHILD_ORDER; break; }
            }
        }
        uint32_t L = 0;
        if (b) {
            bad[i] = b;
        } else if (nd.child_count) {
            // frames: node, its child range, next child, best child level + 1 so far
            uint32_t f_node[kDfsDepth], f_cb[kDfsDepth], f_cc[kDfsDepth], f_k[kDfsDepth], f_best[kDfsDepth];
            int sp = 0;
            uint32_t visits = 0;
            f_node[0] = i; f_cb[0] = nd.child_begin; f_cc[0] = nd.child_count; f_k[0] = 0; f_best[0] = 0;
            sp = 1;
            while (sp > 0) {
                const int t = sp - 1;
                if (f_k[t] < f_cc[t]) {
                    const uint32_t c = __ldg(kids + f_cb[t] + f_k[t]++);
                    const hedl_node cn = nodes[c];
                    const bool valid = c < f_node[t] && (uint64_t)cn.child_begin + cn.child_count <= n_kids;
                    if (!valid || !cn.child_count) {          // a leaf (or an invalid child: its own
                        f_best[t] = max(f_best[t], 1u);       // thread reports it)
                    } else if (sp == kDfsDepth || ++visits > kDfsVisits) {
                        again = true;                         // too deep / too shared: lower bound
                        f_best[t] = max(f_best[t], 1u);
                    } else {
                        f_node[sp] = c; f_cb[sp] = cn.child_begin; f_cc[sp] = cn.child_count; f_k[sp] = 0; f_best[sp] = 0;
                        ++sp;
                    }
                } else {
                    const uint32_t lv = f_best[t];
                    --sp;
                    if (sp > 0) f_best[sp - 1] = max(f_best[sp - 1], lv + 1);
                    else L = lv;
                }
            }
        }
        lvl[i] = L;
        lmax = L;
    }
    if (__any_sync(0xffffffffu, again) && (threadIdx.x & 31) == 0) cnt->changed = 1;
    lmax = __reduce_max_sync(0xffffffffu, lmax);
    if ((threadIdx.x & 31) == 0 && lmax) atomicMax(&cnt->lvl_max, lmax);
}

// level histogram and scatter with block-level aggregation (few distinct levels: global
// atomics on one counter per level would serialise millions of updates)
__global__ void __launch_bounds__(1024) k_dc_hist(const uint32_t *__restrict__ lvl, uint32_t n, uint32_t *hist,
                                                  uint32_t nkeys) {
    extern __shared__ uint32_t sh[];
    for (uint32_t k = threadIdx.x; k < nkeys; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) atomicAdd(sh + lvl[i], 1u);
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < nkeys; k += blockDim.x)
        if (sh[k]) atomicAdd(hist + k, sh[k]);
}

__global__ void __launch_bounds__(1024) k_dc_scatter(const uint32_t *__restrict__ lvl, uint32_t n, uint32_t *cursor,
                                                     uint32_t *list, uint32_t nkeys) {
    extern __shared__ uint32_t sh[];          // [nkeys] local counts, then [nkeys] global bases
    for (uint32_t k = threadIdx.x; k < 2 * nkeys; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t key = 0, r = 0;
    if (i < n) {
        key = lvl[i];
        r = atomicAdd(sh + key, 1u);
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < nkeys; k += blockDim.x)
        if (sh[k]) sh[nkeys + k] = atomicAdd(cursor + k, sh[k]);
    __syncthreads();
    if (i < n) list[sh[nkeys + key] + r] = i;
}

// ---- 2. reachability ------------------------------------------------------------------
__global__ void k_dc_roots_mark(const uint32_t *__restrict__ roots, uint32_t n_roots, uint32_t n, uint8_t *reach,
                                DcCounters *cnt) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_roots) return;
    const uint32_t x = roots[r];
    if (x >= n) dc_error(cnt, r, DE_ROOT_RANGE);
    else reach[x] = 1;
}

__global__ void k_dc_reach(const uint32_t *__restrict__ list, uint32_t m, const hedl_node *__restrict__ nodes,
                           const uint32_t *__restrict__ kids, const uint8_t *__restrict__ bad, uint8_t *reach) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t i = list[t];
    if (!reach[i] || bad[i]) return;
    const hedl_node nd = nodes[i];
    for (uint32_t k = 0; k < nd.child_count; ++k) reach[kids[nd.child_begin + k]] = 1;
}

// ---- 3. validation (reachable nodes) -----------------------------------------------------
__global__ void k_dc_validate(const hedl_node *__restrict__ nodes, uint32_t n, const uint8_t *__restrict__ reach,
                              const uint8_t *__restrict__ bad, DcKb kb, DcCounters *cnt) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !reach[i]) return;
    if (bad[i]) { dc_error(cnt, i, bad[i]); return; }
    const hedl_node nd = nodes[i];
    const uint32_t cc = nd.child_count;
    const bool is_role = nd.op >= HEDL_OP_EXISTS && nd.op <= HEDL_OP_EXACT;
    uint32_t e = DE_NONE;
    if (nd.op == HEDL_OP_SEQUAL || nd.op == HEDL_OP_SCONTAIN) e = DE_STRING;
    else if (nd.op > HEDL_OP_DRANGE) e = DE_OPCODE;
    else if (nd.flags & ~HEDL_FLAG_INV) e = DE_FLAGS;
    else if ((nd.flags & HEDL_FLAG_INV) && !is_role) e = DE_INV_NONROLE;
    else switch (nd.op) {
        case HEDL_OP_TOP: case HEDL_OP_BOTTOM: if (cc) e = DE_ARITY_LEAF; break;
        case HEDL_OP_ATOM: if (cc) e = DE_ARITY_LEAF; else if (nd.arg >= kb.C) e = DE_ATOM_RANGE; break;
        case HEDL_OP_NOT: if (cc != 1) e = DE_ARITY_NOT; break;
        case HEDL_OP_AND: case HEDL_OP_OR: break;
        case HEDL_OP_DRANGE:
            if (cc) e = DE_ARITY_LEAF;
            else if (isnan(nd.lo) || isnan(nd.hi)) e = DE_NAN;
            else if (nd.arg >= kb.D) e = DE_DATA_RANGE;
            break;
        default:
            if (cc != 1) e = DE_ARITY_ROLE;
            else if (nd.arg >= kb.R) e = DE_ROLE_RANGE;
            else if (nd.n > 0xfffffffeu) e = DE_N_BIG;
    }
    if (e) dc_error(cnt, i, e);
}

// ---- 4. canonicalisation + interning ------------------------------------------------------
struct DcOut {
    CNode *nodes;
    uint32_t *ops;
    uint32_t node_cap;
    uint64_t ops_cap;
    uint32_t *table;
    uint64_t mask;
    bool cse, rewrite;
    DcCounters *cnt;
};

__device__ double d_node_bytes(const DcKb &kb, const CNode &n) {
    const double w = 4.0 * kb.W;
    if (n.kind == NK_AND || n.kind == NK_OR) return (n.op_count + 1) * w;
    if (n.kind == NK_RESTRICT) return kb.dir_bytes[n.dir] + 2 * w;
    return kb.data_bytes[n.dir] + w;
}

__device__ uint32_t d_materialise(const DcOut &o, const DcKb &kb, CNode n, const uint32_t *ops, uint64_t node_err) {
    uint32_t lvl = 0;
    bool has_node = false;
    for (uint32_t q = 0; q < n.op_count; ++q)
        if (((ops[q] >> 1) & 3u) == RT_NODE) {
            has_node = true;
            lvl = max(lvl, o.nodes[ops[q] >> 3].level);
        }
    n.level = has_node ? lvl + 1 : 0;
    // id, operand slots and the level maximum for every lane materialising now: one
    // atomic each per warp (millions of same-address atomics would serialise in L2)
    const uint32_t m = __activemask(), lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    const uint32_t below = m & ((1u << lane) - 1u);
    uint32_t opre = 0, otot = 0;
    for (uint32_t mm = m; mm; mm &= mm - 1) {
        const uint32_t l = __ffs(mm) - 1;
        const uint32_t c = __shfl_sync(m, n.op_count, l);
        if (below & (1u << l)) opre += c;
        otot += c;
    }
    const uint32_t lmax = __reduce_max_sync(m, n.level);
    uint32_t idb = 0;
    unsigned long long obb = 0;
    if (lane == leader) {
        idb = atomicAdd(&o.cnt->n_nodes, (uint32_t)__popc(m));
        obb = atomicAdd(&o.cnt->n_ops, (unsigned long long)otot);
        atomicMax(&o.cnt->max_level, lmax);
    }
    const uint32_t id = __shfl_sync(m, idb, leader) + __popc(below);
    const unsigned long long ob = __shfl_sync(m, obb, leader) + opre;
    if (id >= o.node_cap || ob + n.op_count > o.ops_cap) {
        dc_error(o.cnt, node_err, DE_OPS_CAP);
        return 0xffffffffu;
    }
    for (uint32_t q = 0; q < n.op_count; ++q) o.ops[ob + q] = ops[q];
    n.op_begin = (uint32_t)ob;
    n.bytes = d_node_bytes(kb, n);
    o.nodes[id] = n;
    __threadfence();                 // content visible before the id is published
    return id;
}

__device__ uint32_t d_intern(const DcOut &o, const DcKb &kb, const CNode &n, const uint32_t *ops, uint64_t node_err) {
    if (!o.cse) return d_materialise(o, kb, n, ops, node_err);
    uint64_t h = d_hash(n, ops) & o.mask;
    uint32_t mine = 0xffffffffu;
    for (;;) {
        cuda::atomic_ref<uint32_t, cuda::thread_scope_device> slot(o.table[h]);
        uint32_t v = slot.load(cuda::memory_order_acquire);
        if (v == 0) {
            if (mine == 0xffffffffu) {
                mine = d_materialise(o, kb, n, ops, node_err);
                if (mine == 0xffffffffu) return 0;
            }
            uint32_t expected = 0;
            if (slot.compare_exchange_strong(expected, mine + 1, cuda::memory_order_acq_rel,
                                             cuda::memory_order_acquire))
                return mine;
            v = expected;
        }
        const CNode &c = o.nodes[v - 1];
        if (d_same(c, o.ops + c.op_begin, n, ops)) {
            if (mine != 0xffffffffu) o.nodes[mine].kind = NK_DEAD_DEV;   // lost the race: a hole
            return v - 1;
        }
        h = (h + 1) & o.mask;
    }
}

__global__ void __launch_bounds__(128) k_dc_canon(const uint32_t *__restrict__ list, uint32_t m,
                                                  const hedl_node *__restrict__ nodes, const uint32_t *__restrict__ kids,
                                                  const uint8_t *__restrict__ reach, uint32_t *cref, DcOut o, DcKb kb,
                                                  uint32_t flags) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t i = list[t];
    if (!reach[i]) return;
    const hedl_node nd = nodes[i];
    const uint32_t *ch = kids + nd.child_begin;
    uint32_t r = 0;
    switch (nd.op) {
    case HEDL_OP_TOP: case HEDL_OP_BOTTOM: r = d_mkref(RT_TOP, 0, nd.op == HEDL_OP_BOTTOM); break;
    case HEDL_OP_ATOM: r = d_mkref(RT_ATOM, nd.arg, 0); break;
    case HEDL_OP_NOT: r = cref[ch[0]] ^ 1u; break;
    case HEDL_OP_AND: case HEDL_OP_OR: {
        const uint8_t kind = nd.op == HEDL_OP_AND ? NK_AND : NK_OR;
        uint32_t buf[kDcMaxOps];
        uint32_t k = 0;
        for (uint32_t j = 0; j < nd.child_count; ++j) {
            const uint32_t cr = cref[ch[j]];
            if (o.rewrite && ((cr >> 1) & 3u) == RT_NODE && !(cr & 1u) && o.nodes[cr >> 3].kind == kind) {
                const CNode &sub = o.nodes[cr >> 3];
                if (k + sub.op_count > kDcMaxOps) { dc_error(o.cnt, i, DE_OPS_LIMIT); return; }
                for (uint32_t q = 0; q < sub.op_count; ++q) buf[k++] = o.ops[sub.op_begin + q];
            } else {
                if (k + 1 > kDcMaxOps) { dc_error(o.cnt, i, DE_OPS_LIMIT); return; }
                buf[k++] = cr;
            }
        }
        if (o.rewrite) {                     // sort + dedupe (insertion sort: k is small)
            for (uint32_t a = 1; a < k; ++a) {
                const uint32_t v = buf[a];
                uint32_t b = a;
                while (b > 0 && buf[b - 1] > v) { buf[b] = buf[b - 1]; --b; }
                buf[b] = v;
            }
            uint32_t u = 0;
            for (uint32_t a = 0; a < k; ++a)
                if (u == 0 || buf[u - 1] != buf[a]) buf[u++] = buf[a];
            k = u;
        }
        if (k == 0) {
            r = d_mkref(RT_TOP, 0, kind == NK_OR);        // empty AND = TOP, empty OR = BOTTOM
        } else if (k == 1 && o.rewrite) {
            r = buf[0];
        } else {
            CNode n{};
            n.kind = kind;
            n.op_count = k;
            r = d_mkref(RT_NODE, d_intern(o, kb, n, buf, i), 0);
        }
        break;
    }
    case HEDL_OP_DRANGE: {
        CNode n{};
        n.kind = NK_DRANGE;
        n.dir = (uint16_t)nd.arg;
        n.lo = nd.lo;
        n.hi = nd.hi;
        r = d_mkref(RT_NODE, d_intern(o, kb, n, nullptr, i), 0);
        break;
    }
    default: {                               // role restrictions (Alg. 4, 6, 7-8)
        CNode n{};
        n.kind = NK_RESTRICT;
        n.dir = (uint16_t)(2 * nd.arg + (nd.flags & HEDL_FLAG_INV ? 1 : 0));
        n.op_count = 1;
        uint32_t child = cref[ch[0]];
        switch (nd.op) {
        case HEDL_OP_EXISTS: n.pred = P_GE; n.n = 1; n.sat = 1; break;
        case HEDL_OP_FORALL: n.pred = P_LE; n.n = 0; n.sat = 1; child ^= 1u; break;
        case HEDL_OP_MIN: n.pred = P_GE; n.n = nd.n; n.sat = nd.n; break;
        case HEDL_OP_MAX: n.pred = (flags & HEDL_COMPILE_COMPAT_PAPER_MAX) ? P_LEP : P_LE; n.n = nd.n; n.sat = nd.n + 1; break;
        default: n.pred = P_EQ; n.n = nd.n; n.sat = nd.n + 1; break;
        }
        r = d_mkref(RT_NODE, d_intern(o, kb, n, &child, i), 0);
    }
    }
    cref[i] = r;
}

// ---- 5. roots -------------------------------------------------------------------------------
__global__ void k_dc_roots(const uint32_t *__restrict__ roots, uint32_t n_roots, const uint32_t *__restrict__ cref,
                           uint32_t *root_node, DcOut o, DcKb kb) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_roots) return;
    const uint32_t ref = cref[roots[r]];
    if (((ref >> 1) & 3u) == RT_NODE && !(ref & 1u)) {
        root_node[r] = ref >> 3;
    } else {                                 // a 1-operand AND materialises atoms, constants, complements
        CNode n{};
        n.kind = NK_AND;
        n.op_count = 1;
        root_node[r] = d_materialise(o, kb, n, &ref, r);
    }
}

inline uint32_t nblk(uint64_t n, uint32_t t) { return (uint32_t)((n + t - 1) / t); }

}  // namespace

void hedl::dc_free_arrays(hedl_program *p) {
    if (p->d_block) pool_give(p->kb, PR_DC_PROG, p->d_block, p->d_block_bytes);
    p->d_block = nullptr;
    p->d_block_bytes = 0;
    p->d_nodes = nullptr;
    p->d_ops = nullptr;
    p->d_root_node = nullptr;
}

namespace {
// the program's three arrays in one pooled block
bool dc_alloc_arrays(hedl_program *p, uint32_t node_cap, uint64_t ops_cap, uint32_t n_roots) {
    Carver c;
    c.take<CNode>(node_cap);
    c.take<uint32_t>(ops_cap);
    c.take<uint32_t>(std::max<uint32_t>(n_roots, 1));
    size_t got = 0;
    void *blk = pool_alloc(p->kb, PR_DC_PROG, c.off, &got);
    if (!blk) return false;
    p->d_block = blk;
    p->d_block_bytes = got;
    Carver d{(char *)blk, 0};
    p->d_nodes = d.take<CNode>(node_cap);
    p->d_ops = d.take<uint32_t>(ops_cap);
    p->d_root_node = d.take<uint32_t>(std::max<uint32_t>(n_roots, 1));
    return true;
}
}  // namespace

extern "C" hedl_status hedl_compile_device(const hedl_kb *kb, const hedl_node *nodes_in, uint32_t n_nodes,
                                           const uint32_t *child_in, uint64_t n_child_idx, const uint32_t *roots_in,
                                           uint32_t n_roots, uint32_t flags, void *stream, hedl_program **out) {
    const bool host_input = flags & HEDL_COMPILE_HOST_INPUT;
    flags &= ~HEDL_COMPILE_HOST_INPUT;
    const hedl_node *nodes = nodes_in;
    const uint32_t *child_idx = child_in, *roots = roots_in;
    if (!kb || !out) return fail(HEDL_ERR_INVALID_ARG, "null kb/out");
    *out = nullptr;
    if ((n_nodes && !nodes) || (n_child_idx && !child_idx) || (n_roots && !roots))
        return fail(HEDL_ERR_INVALID_ARG, "null node/child/root array");
    if (n_nodes >= (1u << 28)) return fail(HEDL_ERR_INVALID_ARG, "too many nodes in one program (max 2^28)");
    if (kb->poisoned) return fail(HEDL_ERR_CUDA, "KB handle is poisoned by an earlier CUDA error");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != kb->device) cudaSetDevice(kb->device);
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};
    const double t0 = now_ms();
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t n = n_nodes;
    const uint32_t node_cap = n + n_roots + 1;
    uint64_t tcap = 1024;
    while (tcap < 2ull * node_cap) tcap <<= 1;
    const bool cse = !(flags & HEDL_COMPILE_NO_CSE);
    // scratch: one pooled block (no cudaMalloc / cudaFree per compile)
    uint32_t *lvl, *list, *cref, *hist, *cursor, *table;
    uint8_t *bad, *reach;
    DcCounters *cnt;
    double *kbytes;
    size_t sgot = 0;
    void *sblk = nullptr;
    for (int pass = 0; pass < 2; ++pass) {
        Carver c{(char *)sblk, 0};
        lvl = c.take<uint32_t>(n);
        list = c.take<uint32_t>(n);
        cref = c.take<uint32_t>(n);
        hist = c.take<uint32_t>(kDcMaxDepth + 3);
        cursor = c.take<uint32_t>(kDcMaxDepth + 3);
        table = c.take<uint32_t>(cse ? tcap : 1);
        bad = c.take<uint8_t>(n);
        reach = c.take<uint8_t>(n);
        cnt = c.take<DcCounters>(1);
        kbytes = c.take<double>(2 * kb->R + kb->D + 1);
        if (host_input) {          // device copies of the caller's host arrays (staged below)
            nodes = c.take<hedl_node>(n);
            child_idx = c.take<uint32_t>(n_child_idx);
            roots = c.take<uint32_t>(n_roots);
        }
        if (pass == 0 && !(sblk = pool_alloc(kb, PR_DC_SCRATCH, c.off, &sgot))) return fail(HEDL_ERR_OOM, "device compile scratch");
    }
    struct GiveBack { const hedl_kb *kb; void *p; size_t b; ~GiveBack() { pool_give(kb, PR_DC_SCRATCH, p, b); } } gb{kb, sblk, sgot};
    // pinned read-back word, one per host thread (no cudaMallocHost per compile)
    struct PinnedCounters {
        DcCounters *p = nullptr;
        ~PinnedCounters() { if (p) cudaFreeHost(p); }
    };
    static thread_local PinnedCounters pinned;
    if (!pinned.p && cudaMallocHost((void **)&pinned.p, sizeof(DcCounters)) != cudaSuccess) {
        cudaGetLastError();
        pinned.p = nullptr;
        return fail(HEDL_ERR_OOM, "pinned");
    }
    DcCounters *hc = pinned.p;
    {   // pageable source: the copy is staged before the call returns
        std::vector<double> kbb(kb->dir_bytes.begin(), kb->dir_bytes.end());
        kbb.insert(kbb.end(), kb->data_bytes.begin(), kb->data_bytes.end());
        kbb.push_back(0);
        HEDL_CUDA(kb, cudaMemcpy(kbytes, kbb.data(), kbb.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    if (host_input) {
        // H2D of the batch on the call's stream: DMA straight from page-locked arrays (the
        // e2e path of bench.py), staged by the driver from pageable ones
        HEDL_CUDA(kb, cudaMemcpyAsync((void *)nodes, nodes_in, (size_t)n * sizeof(hedl_node), cudaMemcpyHostToDevice, s));
        HEDL_CUDA(kb, cudaMemcpyAsync((void *)child_idx, child_in, n_child_idx * 4, cudaMemcpyHostToDevice, s));
        HEDL_CUDA(kb, cudaMemcpyAsync((void *)roots, roots_in, (size_t)n_roots * 4, cudaMemcpyHostToDevice, s));
        count_io((size_t)n * sizeof(hedl_node) + n_child_idx * 4 + (size_t)n_roots * 4, 0);
    }
    const DcKb dk{kb->C, kb->R, kb->D, kb->W, kbytes, kbytes + 2 * kb->R};
    DcCounters init{0, 0, 0, ~0ull, 0, 0};
    HEDL_CUDA(kb, cudaMemcpyAsync(cnt, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    HEDL_CUDA(kb, cudaMemsetAsync(lvl, 0, (size_t)n * 4, s));
    HEDL_CUDA(kb, cudaMemsetAsync(bad, 0, n, s));
    HEDL_CUDA(kb, cudaMemsetAsync(reach, 0, n, s));
    auto read_counters = [&]() -> hedl_status {
        HEDL_CUDA(kb, cudaMemcpyAsync(hc, cnt, sizeof(DcCounters), cudaMemcpyDeviceToHost, s));
        HEDL_CUDA(kb, cudaStreamSynchronize(s));
        return HEDL_OK;
    };
    auto report = [&]() -> hedl_status {
        if (hc->err == ~0ull) return HEDL_OK;
        const uint32_t code = (uint32_t)(hc->err & 0xff);
        const uint64_t at = hc->err >> 8;
        const DcErrInfo &e = kDcErr[code < sizeof(kDcErr) / sizeof(kDcErr[0]) ? code : 0];
        return fail(e.st, (code == DE_ROOT_RANGE ? "root " : "node ") + std::to_string(at) + ": " + e.msg);
    };
    hedl_status st;
    // 1. levels: one bounded depth-first pass; relaxation passes only if it ran out of budget
    if (n) k_dc_level_dfs<<<nblk(n, 256), 256, 0, s>>>(nodes, n, child_idx, n_child_idx, lvl, bad, cnt);
    count_launch();
    if ((st = read_counters())) return st;
    for (uint32_t depth = 0; hc->changed; ++depth) {
        if (depth > kDcMaxDepth) return fail(kDcErr[DE_DEPTH].st, kDcErr[DE_DEPTH].msg);
        HEDL_CUDA(kb, cudaMemsetAsync(&cnt->changed, 0, 4, s));
        if (n) k_dc_level<<<nblk(n, 256), 256, 0, s>>>(nodes, n, child_idx, n_child_idx, lvl, bad, cnt);
        count_launch();
        if ((st = read_counters())) return st;
    }
    timing_note("device compile: levels", now_ms() - t0);
    const uint32_t L = hc->lvl_max + 1;   // levels 0 .. lvl_max occur
    // 2. level lists, reachability (top-down)
    HEDL_CUDA(kb, cudaMemsetAsync(hist, 0, (L + 1) * 4, s));
    if (n) k_dc_hist<<<std::min<uint32_t>(nblk(n, 1024), 1184), 1024, (L + 1) * 4, s>>>(lvl, n, hist, L + 1);
    std::vector<uint32_t> h_hist(L + 1), h_off(L + 2, 0);
    HEDL_CUDA(kb, cudaMemcpyAsync(h_hist.data(), hist, (L + 1) * 4, cudaMemcpyDeviceToHost, s));
    HEDL_CUDA(kb, cudaStreamSynchronize(s));
    for (uint32_t l = 0; l <= L; ++l) h_off[l + 1] = h_off[l] + h_hist[l];
    HEDL_CUDA(kb, cudaMemcpyAsync(cursor, h_off.data(), (L + 1) * 4, cudaMemcpyHostToDevice, s));
    if (n) k_dc_scatter<<<nblk(n, 1024), 1024, 2 * (L + 1) * 4, s>>>(lvl, n, cursor, list, L + 1);
    if (n_roots) k_dc_roots_mark<<<nblk(n_roots, 256), 256, 0, s>>>(roots, n_roots, n, reach, cnt);
    for (uint32_t l = L + 1; l-- > 1;)
        if (h_hist[l]) k_dc_reach<<<nblk(h_hist[l], 256), 256, 0, s>>>(list + h_off[l], h_hist[l], nodes, child_idx, bad, reach);
    // 3. validation
    if (n) k_dc_validate<<<nblk(n, 256), 256, 0, s>>>(nodes, n, reach, bad, dk, cnt);
    if ((st = read_counters())) return st;
    if ((st = report())) return st;
    timing_note("device compile: reach+validate", now_ms() - t0);
    // 4. canonicalisation, level by level up; 5. roots
    hedl_program *p = new hedl_program();
    p->kb = kb;
    p->flags = flags;
    p->dev = true;
    p->root_node.clear();
    uint64_t ops_cap = 2 * n_child_idx + n_roots + 1024;
    for (int attempt = 0; attempt < 2; ++attempt) {
        dc_free_arrays(p);
        if (!dc_alloc_arrays(p, node_cap, ops_cap, n_roots)) {
            delete p;
            return fail(HEDL_ERR_OOM, "device program arrays");
        }
        HEDL_CUDA(kb, cudaMemcpyAsync(cnt, &init, sizeof(init), cudaMemcpyHostToDevice, s));
        if (cse) HEDL_CUDA(kb, cudaMemsetAsync(table, 0, tcap * 4, s));
        const DcOut o{p->d_nodes, p->d_ops, node_cap, ops_cap, table, tcap - 1, cse, !(flags & HEDL_COMPILE_NO_REWRITE), cnt};
        for (uint32_t l = 0; l <= L; ++l)
            if (h_hist[l]) {
                k_dc_canon<<<nblk(h_hist[l], 128), 128, 0, s>>>(list + h_off[l], h_hist[l], nodes, child_idx, reach, cref,
                                                                o, dk, flags);
                count_launch();
            }
        if (n_roots) k_dc_roots<<<nblk(n_roots, 256), 256, 0, s>>>(roots, n_roots, cref, p->d_root_node, o, dk);
        if ((st = read_counters())) { dc_free_arrays(p); delete p; return st; }
        if (hc->err != ~0ull && (hc->err & 0xff) == DE_OPS_CAP && attempt == 0) {
            ops_cap = std::max<uint64_t>(ops_cap * 2, hc->n_ops + 1024);   // flattening grew the operand table
            continue;
        }
        break;
    }
    if ((st = report())) { dc_free_arrays(p); delete p; return st; }
    p->dev_n_nodes = std::min(hc->n_nodes, node_cap);
    p->dev_n_ops = hc->n_ops;
    p->dev_n_roots = n_roots;
    p->n_levels = p->dev_n_nodes ? hc->max_level + 1 : 0;
    const_cast<hedl_kb *>(kb)->refs.fetch_add(1);        // released by hedl_program_free
    timing_note("device compile: total", now_ms() - t0);
    *out = p;
    return HEDL_OK;
}

namespace hedl {
// Host copy of a device-compiled program (nodes, operands, roots): lets the host-side
// utilities (info, root bytes, the latency interpreter) read it.
hedl_status dc_download(hedl_program *p) {
    if (!p->dev || p->dev_downloaded) return HEDL_OK;
    const hedl_kb *kb = p->kb;
    p->nodes.resize(p->dev_n_nodes);
    p->ops.resize(p->dev_n_ops);
    p->root_node.resize(p->dev_n_roots);
    HEDL_CUDA(kb, cudaMemcpy(p->nodes.data(), p->d_nodes, (size_t)p->dev_n_nodes * sizeof(CNode), cudaMemcpyDeviceToHost));
    HEDL_CUDA(kb, cudaMemcpy(p->ops.data(), p->d_ops, p->dev_n_ops * 4, cudaMemcpyDeviceToHost));
    HEDL_CUDA(kb, cudaMemcpy(p->root_node.data(), p->d_root_node, (size_t)p->dev_n_roots * 4, cudaMemcpyDeviceToHost));
    p->stamp.assign(p->nodes.size(), 0);
    p->dev_downloaded = true;
    return HEDL_OK;
}
}  // namespace hedl

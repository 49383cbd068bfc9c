// Executor: hedl_eval_one / hedl_eval_batch.
//
// A set of roots is planned as one or more chunks.  Per chunk the needed
// canonical nodes are collected, grouped by topological level and then by
// (kind, role direction / data property), and each group runs as ONE launch
// whose blockIdx.y walks the group's nodes (consecutive nodes of one direction
// re-hit the same CSR in L2); restriction groups of >= kSliceMinNodes nodes run
// as lane-packed passes (slice.cu).  Root nodes fuse the Alg. 15 coverage
// (PAPER.md:548-553).  The plan (descriptors of every launch) is the paper's
// "evaluation plan": built on the first call for a root range,
// kept device-resident in the program, and replayed by later calls.  Counts come
// back with one D2H per call (the paper's single cudaMemcpyAsync).
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <thread>

#include "exec.h"
#include "interp.h"
#include "slice.h"

using namespace hedl;

namespace hedl {

Workspace *ws_of(hedl_program *p) {
    if (!p->ws) p->ws = new Workspace();
    return (Workspace *)p->ws;
}

// a sub-block of the caller's workspace (hedl_program_set_workspace); OOM when it is full
static hedl_status carve(const hedl_kb *kb, cudaStream_t s, Workspace *w, void **p, size_t need, bool zero) {
    const size_t a = align_up(need, 256);
    if (w->ext_used + a > w->ext_bytes)
        return fail(HEDL_ERR_OOM, "caller workspace too small (" + std::to_string(w->ext_bytes) +
                                      " bytes; hedl_program_workspace_bytes gives the need)");
    *p = w->ext + w->ext_used;
    w->ext_used += a;
    if (zero) HEDL_CUDA(kb, cudaMemsetAsync(*p, 0, need, s));
    return HEDL_OK;
}

hedl_status grow(const hedl_kb *kb, cudaStream_t s, DevBuf &b, size_t need, bool zero, int role, Workspace *w) {
    if (b.bytes >= need) return HEDL_OK;
    if (w && w->ext) {
        hedl_status st = carve(kb, s, w, &b.p, need, zero);
        b.bytes = st ? 0 : need;
        if (st) b.p = nullptr;
        return st;
    }
    if (b.p) HEDL_CUDA(kb, cudaStreamSynchronize(s));  // the old buffer may still be in use
    size_t sz = std::max(need, b.bytes * 5 / 4);
    if (b.p) dev_free(b.p, s);
    b.p = nullptr;
    b.bytes = 0;
    size_t got = 0;
    if (void *q = pool_take(kb, role, need, &got)) {   // pooled buffers come back self-cleaned
        b.p = q;
        b.bytes = got;
        return HEDL_OK;
    }
    sz = (sz + 255) & ~size_t(255);
    cudaError_t e = dev_malloc(&b.p, sz, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        e = dev_malloc(&b.p, need, s);
        if (e != cudaSuccess) { cudaGetLastError(); b.p = nullptr; return fail(HEDL_ERR_OOM, "workspace allocation failed"); }
        sz = need;
    }
    b.bytes = sz;
    if (zero) HEDL_CUDA(kb, cudaMemsetAsync(b.p, 0, sz, s));
    return HEDL_OK;
}

void drop_graph(PlanCache &pc) {
    if (pc.graph) cudaGraphExecDestroy(pc.graph);
    pc.graph = nullptr;
    pc.g_counts = pc.g_bits = nullptr;
    pc.g_calls = 0;
}

void invalidate_plan(PlanCache &pc) {
    pc.valid = false;
    pc.chunks.clear();
    drop_graph(pc);
}

// Replays of a cached plan go through a CUDA graph of its launches (captured on the second
// replay with the same output buffers; the plan's descriptors, workspace and outputs are all
// fixed addresses then), on the library's own stream between two events.  Not while library
// profiling is on (its events are per launch), not with HEDL_NO_GRAPH set; a failed capture
// falls back to plain launches on the caller's stream.
hedl_status replay_plan(const hedl_kb *kb, Workspace *w, uint32_t r0, uint32_t *out_bits, hedl_counts *counts_dev,
                        cudaStream_t s) {
    PlanCache &pc = w->plan;
    static const bool no_graph = std::getenv("HEDL_NO_GRAPH") != nullptr;
    hedl_status st = HEDL_OK;
    auto direct = [&](cudaStream_t on) -> hedl_status {
        for (const ChunkPlan &cp : pc.chunks)
            if ((st = launch_chunk(kb, w, cp, r0, out_bits, counts_dev, on))) return st;
        return HEDL_OK;
    };
    if (no_graph || prof_active()) return direct(s);
    if (pc.g_counts != counts_dev || pc.g_bits != out_bits) {
        drop_graph(pc);
        pc.g_counts = counts_dev;
        pc.g_bits = out_bits;
    }
    if (!pc.graph && ++pc.g_calls < 2) return direct(s);    // capture once the outputs repeat
    if (!pc.gstream) {
        if (cudaStreamCreateWithFlags(&pc.gstream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&pc.gev_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&pc.gev_out, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            return direct(s);
        }
    }
    HEDL_CUDA(kb, cudaEventRecord(pc.gev_in, s));
    HEDL_CUDA(kb, cudaStreamWaitEvent(pc.gstream, pc.gev_in, 0));
    if (!pc.graph) {
        cudaGraph_t g = nullptr;
        if (cudaStreamBeginCapture(pc.gstream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            cudaGetLastError();
            return direct(s);
        }
        const uint64_t l0 = launches_total();
        const hedl_status cs = direct(pc.gstream);
        const cudaError_t ce = cudaStreamEndCapture(pc.gstream, &g);
        pc.g_launches = launches_total() - l0;
        cudaGraphExec_t ex = nullptr;
        const bool ok = !cs && ce == cudaSuccess && g && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        if (!ok) {
            cudaGetLastError();
            pc.g_calls = 0;
            return direct(s);
        }
        pc.graph = ex;
    } else {
        count_launches(pc.g_launches);
    }
    HEDL_CUDA(kb, cudaGraphLaunch(pc.graph, pc.gstream));
    HEDL_CUDA(kb, cudaEventRecord(pc.gev_out, pc.gstream));
    HEDL_CUDA(kb, cudaStreamWaitEvent(s, pc.gev_out, 0));
    return HEDL_OK;
}

void release_plan(PlanCache &pc) {
    drop_graph(pc);
    if (pc.gstream) cudaStreamDestroy(pc.gstream);
    if (pc.gev_in) cudaEventDestroy(pc.gev_in);
    if (pc.gev_out) cudaEventDestroy(pc.gev_out);
    if (pc.host) cudaFreeHost(pc.host);
    if (pc.dev) dev_free(pc.dev);
    pc = PlanCache();
}

hedl_status reserve_plan(const hedl_kb *kb, PlanCache &pc, size_t bytes, Workspace *w) {
    if (pc.cap >= bytes) return HEDL_OK;
    if (w && w->ext) {      // device blob from the caller's block, pinned host blob from the library
        const size_t cap = std::max(bytes, (size_t)4096);
        if (pc.host_cap < cap) {
            if (pc.host) cudaFreeHost(pc.host);
            pc.host = nullptr;
            pc.host_cap = 0;
            if (cudaMallocHost(&pc.host, cap * 5 / 4) != cudaSuccess) { cudaGetLastError(); pc.host = nullptr; return fail(HEDL_ERR_OOM, "pinned plan"); }
            pc.host_cap = cap * 5 / 4;
        }
        pc.dev = nullptr;
        pc.cap = 0;
        hedl_status st = carve(kb, nullptr, w, &pc.dev, cap, false);
        if (st) return st;
        pc.cap = cap;
        return HEDL_OK;
    }
    if (pc.host) cudaFreeHost(pc.host);
    if (pc.dev) dev_free(pc.dev);
    pc.host = pc.dev = nullptr;
    pc.cap = 0;
    size_t gh = 0, gd = 0;
    void *h = pool_take(kb, PR_PLAN_HOST, bytes, &gh);
    void *d = pool_take(kb, PR_PLAN_DEV, bytes, &gd);
    if (h && d) {
        pc.host = h;
        pc.dev = d;
        pc.cap = std::min(gh, gd);
        return HEDL_OK;
    }
    // a pooled half is kept; only the missing one is allocated
    size_t cap = std::max(bytes, (size_t)4096) * 5 / 4;
    if (h) {
        pc.host = h;
        cap = std::min(cap, gh);
    } else {
        if (d) cap = std::min(cap, gd);
        const double t0 = now_ms();
        if (cudaMallocHost(&pc.host, cap) != cudaSuccess) {
            cudaGetLastError();
            pc.host = nullptr;
            if (d) pool_give(kb, PR_PLAN_DEV, d, gd);
            return fail(HEDL_ERR_OOM, "pinned plan");
        }
        timing_note("plan: cudaMallocHost", now_ms() - t0);
    }
    if (d) {
        pc.dev = d;
    } else if (dev_malloc(&pc.dev, cap) != cudaSuccess) {
        cudaGetLastError();
        pool_give(kb, PR_PLAN_HOST, pc.host, cap);
        pc.host = pc.dev = nullptr;
        return fail(HEDL_ERR_OOM, "device plan");
    }
    pc.cap = cap;
    return HEDL_OK;
}

}  // namespace hedl

namespace {


struct Group {
    uint8_t kind;
    uint16_t key;
    uint32_t first, count;   // into ChunkTmp::members (positions in the chunk list)
    bool slice = false;
    bool proj = false;
    bool ex = false;
    int16_t usp = -1;        // boolean group evaluated over U of direction usp
    bool ucomp = false;      // EX pack whose fillers are U rows
    int8_t usw = -1;         // U-sweep pack: rows of U_usw only, results to U rows
};

// ---- planning (host threads, as the paper generates plans in parallel) ----
unsigned plan_threads() {
    static const unsigned t = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    return t;
}

// f(begin, end) over [0, n) in chunks of `grain`, dynamically scheduled over host threads
template <class F>
void par_for(size_t n, size_t grain, F f) {
    const unsigned T = (unsigned)std::min<size_t>(plan_threads(), (n + grain - 1) / std::max<size_t>(grain, 1));
    if (T <= 1) { if (n) f((size_t)0, n); return; }
    std::atomic<size_t> next{0};
    auto work = [&]() {
        for (;;) {
            const size_t b = next.fetch_add(grain);
            if (b >= n) break;
            f(b, std::min(n, b + grain));
        }
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back(work);
    work();
    for (auto &x : th) x.join();
}

// out[k] = rank of k among the k' < k with flag(k') (for flagged k); returns the count
template <class Flag, class Out>
uint32_t par_rank(size_t n, Flag flag, Out &out) {
    if (n < (1u << 15)) {                          // small plans: no thread start-up
        uint32_t r = 0;
        for (size_t k = 0; k < n; ++k)
            if (flag(k)) out[k] = r++;
        return r;
    }
    const size_t C = 64;
    std::vector<uint32_t> cnt(C + 1, 0);
    par_for(C, 1, [&](size_t c0, size_t c1) {
        for (size_t c = c0; c < c1; ++c)
            for (size_t k = n * c / C; k < n * (c + 1) / C; ++k) cnt[c + 1] += flag(k) ? 1u : 0u;
    });
    for (size_t c = 0; c < C; ++c) cnt[c + 1] += cnt[c];
    par_for(C, 1, [&](size_t c0, size_t c1) {
        for (size_t c = c0; c < c1; ++c) {
            uint32_t r = cnt[c];
            for (size_t k = n * c / C; k < n * (c + 1) / C; ++k)
                if (flag(k)) out[k] = r++;
        }
    });
    return cnt[C];
}

// order key: level, kind, direction / property / string role, lane-pack class (node id breaks ties)
inline uint64_t group_key(const CNode &n) {
    const uint32_t cls = n.kind == NK_RESTRICT ? slice_class(n.pred, n.n, n.sat) : 0;
    const uint32_t kind = n.kind == NK_OR ? NK_AND : n.kind;
    return ((uint64_t)n.level << 24) | ((uint64_t)(kind & 7) << 20) | ((uint64_t)n.dir << 2) | cls;
}

// stable bucket sort of `list` (ascending ids) by group_key: parallel histogram + scatter
void sort_by_key(const hedl_program *p, std::vector<uint32_t> &list) {
    const size_t n = list.size();
    if (n < (1u << 15)) {
        std::stable_sort(list.begin(), list.end(), [&](uint32_t a, uint32_t b) {
            return group_key(p->nodes[a]) < group_key(p->nodes[b]);
        });
        return;
    }
    std::vector<uint64_t> key(n);
    par_for(n, 1 << 14, [&](size_t a, size_t b) { for (size_t k = a; k < b; ++k) key[k] = group_key(p->nodes[list[k]]); });
    std::vector<uint64_t> uk;                      // distinct keys (few: levels x kinds x directions x classes)
    {
        std::vector<uint64_t> tmp;
        for (size_t k = 0; k < n; k += 97) tmp.push_back(key[k]);
        std::sort(tmp.begin(), tmp.end());
        tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
        uk = tmp;
        for (size_t k = 0; k < n; ++k)
            if (!std::binary_search(uk.begin(), uk.end(), key[k])) {
                uk.insert(std::upper_bound(uk.begin(), uk.end(), key[k]), key[k]);
            }
    }
    const size_t B = uk.size(), C = 64;            // C contiguous chunks of the list
    std::vector<uint32_t> bk(n);
    std::vector<uint64_t> hist(C * B, 0);
    par_for(C, 1, [&](size_t c0, size_t c1) {
        for (size_t c = c0; c < c1; ++c) {
            const size_t a = n * c / C, b = n * (c + 1) / C;
            for (size_t k = a; k < b; ++k) {
                bk[k] = (uint32_t)(std::lower_bound(uk.begin(), uk.end(), key[k]) - uk.begin());
                hist[c * B + bk[k]]++;
            }
        }
    });
    std::vector<uint64_t> off(C * B);
    uint64_t acc = 0;
    for (size_t b = 0; b < B; ++b)
        for (size_t c = 0; c < C; ++c) { off[c * B + b] = acc; acc += hist[c * B + b]; }
    std::vector<uint32_t> out(n);
    par_for(C, 1, [&](size_t c0, size_t c1) {
        for (size_t c = c0; c < c1; ++c) {
            const size_t a = n * c / C, b = n * (c + 1) / C;
            uint64_t *o = &off[c * B];
            for (size_t k = a; k < b; ++k) out[o[bk[k]]++] = list[k];
        }
    });
    list.swap(out);
}

// Phase A: the node list of every chunk (host only).  Rows are materialised only
// for nodes some other node reads, so the row budget counts operand nodes.
void collect_chunks(hedl_program *p, uint32_t r0, uint32_t r1, uint64_t row_cap,
                    std::vector<std::vector<uint32_t>> &lists, std::vector<std::pair<uint32_t, uint32_t>> &ranges) {
    if (p->stamp.size() < p->nodes.size()) p->stamp.assign(p->nodes.size(), 0);
    if (r0 == 0 && r1 == p->root_node.size()) {
        // the whole program: every live node is reachable from a root
        const size_t NN = p->nodes.size(), C = NN < (1u << 15) ? 1 : 64;
        std::vector<uint32_t> cnt(C + 1, 0);
        par_for(C, 1, [&](size_t c0, size_t c1) {
            for (size_t c = c0; c < c1; ++c)
                for (size_t i = NN * c / C; i < NN * (c + 1) / C; ++i) cnt[c + 1] += p->nodes[i].kind <= NK_STRING;
        });
        for (size_t c = 0; c < C; ++c) cnt[c + 1] += cnt[c];
        const uint64_t live = cnt[C];
        if (live - std::min<uint64_t>(live, r1) <= row_cap) {
            std::vector<uint32_t> list(live);
            par_for(C, 1, [&](size_t c0, size_t c1) {
                for (size_t c = c0; c < c1; ++c) {
                    uint32_t o = cnt[c];
                    for (size_t i = NN * c / C; i < NN * (c + 1) / C; ++i)
                        if (p->nodes[i].kind <= NK_STRING) list[o++] = (uint32_t)i;
                }
            });
            sort_by_key(p, list);
            lists.push_back(std::move(list));
            ranges.push_back({r0, r1});
            return;
        }
    }
    std::vector<uint32_t> st;
    uint32_t ri = r0;
    while (ri < r1) {
        const uint32_t gen = ++p->stamp_gen;
        std::vector<uint32_t> list;
        uint64_t operands = 0;
        uint32_t rc = ri;
        for (; rc < r1; ++rc) {
            const size_t before = list.size();
            const uint64_t ob = operands;
            if (p->stamp[p->root_node[rc]] == gen) continue;
            p->stamp[p->root_node[rc]] = gen;
            st.assign(1, p->root_node[rc]);
            while (!st.empty()) {
                const uint32_t id = st.back();
                st.pop_back();
                list.push_back(id);
                const CNode &n = p->nodes[id];
                for (uint32_t q = 0; q < n.op_count; ++q) {
                    const uint32_t o = p->ops[n.op_begin + q];
                    if (ref_type(o) == RT_NODE && p->stamp[ref_id(o)] != gen) {
                        p->stamp[ref_id(o)] = gen;
                        st.push_back(ref_id(o));
                        ++operands;
                    }
                }
            }
            if (operands > row_cap && rc > ri) {    // this root overflows the chunk: defer it
                for (size_t k = before; k < list.size(); ++k) p->stamp[list[k]] = 0;
                list.resize(before);
                operands = ob;
                break;
            }
        }
        sort_by_key(p, list);
        lists.push_back(std::move(list));
        ranges.push_back({ri, rc});
        ri = rc;
    }
}

struct ChunkTmp {            // per-chunk planning state kept between the sizing and filling passes
    std::vector<uint32_t> slot, pslot, cover_of_root, members, gdesc, opbase;
    std::vector<int32_t> cover_of_node;
    std::vector<uint8_t> need_full, need_proj, pmode;
    // boolean fillers fused into the packs: a full row only lane packs
    // read is never materialised; the pack kernel combines the node's operand rows itself
    std::vector<uint8_t> by_pack, by_other, fused;
    std::vector<int8_t> uswd;          // U-sweep direction of a restriction (-1: full pack / EX / per-node)
    std::vector<uint64_t> need_u;      // directions whose U rows of the node are read
    std::vector<uint64_t> u_out;       // directions whose U rows the node (a boolean) computes
    std::vector<uint32_t> ubase;       // first U-row slot of the node
    std::vector<Group> groups;
};

// Phase C: descriptors of one chunk into `h` (host blob) with device addresses.
// Called twice: sizes_only (fills tmp and the blob layout), then with the final buffers.
//
// Example projection: coverage only reads bits at P u N.  A boolean
// node nobody needs in full (e.g. a root conjunction) runs on example-projected
// rows (M bits instead of N); its operands then only need projected rows, which
// atoms/TOP have precomputed and computed nodes emit as a scatter epilogue.
void fill_chunk(const hedl_kb *kb, hedl_program *p, const std::vector<uint32_t> &list, ChunkPlan &cp,
                bool out_bits, bool use_slice, bool force_slice, bool allow_fuse, bool allow_urestr, bool allow_usw, uint32_t *rows, uint32_t *prows, uint32_t *urows,
                std::vector<uint32_t> &local, char *h_blob, size_t *blob_cursor, size_t *heavy_need, bool sizes_only,
                ChunkTmp &tmp) {
    const uint32_t nn = (uint32_t)list.size();
    cp.nn = nn;
    par_for(nn, 1 << 15, [&](size_t a, size_t b) { for (size_t k = a; k < b; ++k) local[list[k]] = (uint32_t)k; });
    const uint32_t nroots = cp.rc - cp.ri;
    auto &need_full = tmp.need_full;
    auto &need_proj = tmp.need_proj;
    auto &pmode = tmp.pmode;
    auto &slot = tmp.slot;
    auto &pslot = tmp.pslot;
    auto &cover_of_node = tmp.cover_of_node;
    auto &cover_of_root = tmp.cover_of_root;
    auto &groups = tmp.groups;
    auto &members = tmp.members;
    if (sizes_only) {
        const double ts0 = now_ms();
        // one count slot per distinct root node
        cover_of_node.assign(nn, -1);
        cover_of_root.resize(nroots);
        std::vector<uint8_t> isroot(nn, 0);
        par_for(nroots, 1 << 15, [&](size_t a, size_t b) {
            for (size_t k = a; k < b; ++k) isroot[local[p->root_node[cp.ri + k]]] = 1;
        });
        const uint32_t ncov = par_rank(nn, [&](size_t k) { return isroot[k] != 0; }, cover_of_node);
        par_for(nroots, 1 << 15, [&](size_t a, size_t b) {
            for (size_t k = a; k < b; ++k) cover_of_root[k] = (uint32_t)cover_of_node[local[p->root_node[cp.ri + k]]];
        });
        cp.ncov = ncov;
        // demands, consumers first (the list is in ascending level order)
        need_full.assign(nn, 0);
        need_proj.assign(nn, 0);
        pmode.assign(nn, 0);
        auto &by_pack = tmp.by_pack;
        auto &by_other = tmp.by_other;
        auto &fused = tmp.fused;
        by_pack.assign(nn, 0);
        by_other.assign(nn, 0);
        fused.assign(nn, 0);
        auto &uswd = tmp.uswd;
        uswd.assign(nn, -1);
        auto &need_u = tmp.need_u;
        auto &u_out = tmp.u_out;
        need_u.assign(nn, 0);
        u_out.assign(nn, 0);
        if (out_bits)
            for (uint32_t k = 0; k < nroots; ++k) need_full[local[p->root_node[cp.ri + k]]] = by_other[local[p->root_node[cp.ri + k]]] = 1;
        // U rows: an EX-pack restriction in direction d reads its
        // filler only at U_d (the example rows' neighbours).  A boolean over atoms / TOP /
        // such booleans ("U-capable") demanded over U_d is evaluated over U_d (a row of |U_d|
        // bits), besides any full or example-projected row it is needed as; other fillers are
        // computed in full and the pack reads their full rows at U_d.
        const bool use_u = use_slice && kb->M > 0;
        // restrictions in full lane packs emit U rows from the tile epilogue (DESIGN.md "U rows
        // of restrictions"), so booleans over them are U-capable too
        const bool u_restr = use_u && allow_urestr && kb->dirs.size() <= kMaxUDirs;
        // a restriction needed only as one U row (not in full, not projected, not a root) is
        // swept over the rows of that U set only
        const bool use_usw = u_restr && allow_usw;
        auto usw_of = [&](size_t kk, uint64_t uo) -> int {
            if (!use_usw || !uo || need_full[kk] || need_proj[kk] || cover_of_node[kk] >= 0) return -1;
            if (__builtin_popcountll(uo) != 1) return -1;
            const CNode &n = p->nodes[list[kk]];
            if (n.kind != NK_RESTRICT || slice_class(n.pred, n.n, n.sat) >= 2) return -1;
            const int d = __builtin_ctzll(uo);
            return (d < (int)kMaxUDirs && kb->dirs[n.dir].usw[d].n_rows) ? d : -1;
        };
        std::vector<uint8_t> ucap(nn, 0);
        if (use_u)
            for (uint32_t lo = 0; lo < nn;) {                  // bottom-up, level by level
                uint32_t hi = lo + 1;
                while (hi < nn && p->nodes[list[hi]].level == p->nodes[list[lo]].level) ++hi;
                par_for(hi - lo, 1 << 13, [&](size_t a, size_t b) {
                    for (size_t kk = lo + a; kk < lo + b; ++kk) {
                        const CNode &n = p->nodes[list[kk]];
                        if (n.kind == NK_RESTRICT) {
                            ucap[kk] = u_restr && slice_class(n.pred, n.n, n.sat) < 2;
                            continue;
                        }
                        if (n.kind == NK_DRANGE) {           // ranges are evaluated at U members directly
                            ucap[kk] = use_u && allow_urestr;
                            continue;
                        }
                        bool c = n.kind == NK_AND || n.kind == NK_OR;
                        for (uint32_t q = 0; c && q < n.op_count; ++q) {
                            const uint32_t o = p->ops[n.op_begin + q];
                            if (ref_type(o) == RT_NODE && !ucap[local[ref_id(o)]]) c = false;
                        }
                        ucap[kk] = c;
                    }
                });
                lo = hi;
            }
        // level by level from the top; within a level nodes are independent (operands sit at
        // lower levels; concurrent writes of 1 to a shared operand flag are benign, U demands
        // are atomic ORs)
        for (uint32_t hi = nn; hi > 0;) {
            const uint32_t lvl = p->nodes[list[hi - 1]].level;
            uint32_t lo = hi - 1;
            while (lo > 0 && p->nodes[list[lo - 1]].level == lvl) --lo;
            // this level's demands are final: restrictions an EX pack reads as full-row fillers
            // are needed in full; then which (level, direction) groups run as full lane packs
            // (the same rule the grouping below applies), so their fillers' demand is a pack's
            // (restrictions emitting U rows run in full packs too, and force their group's packing)
            uint32_t nfull_dir[64] = {0};
            uint64_t uforce = 0;
            // U sweeps: per (direction, class) the candidates of each U set
            // either get packs of their own (rows of U_d only) or join the full packs; the cheaper
            // split by a per-pack cost model (full pack: T build + heavy rows + full sweep = 1.42;
            // U pack: T build + heavy / sweep at the U set's edge fraction f = 0.20 + 1.22 f)
            if (use_usw) {
                uint32_t F[64][2] = {{0}}, Lc[64][2][kMaxUDirs] = {{{0}}};
                for (uint32_t kk = lo; kk < hi; ++kk) {
                    const CNode &n = p->nodes[list[kk]];
                    if (n.kind != NK_RESTRICT) continue;
                    const uint32_t cls = slice_class(n.pred, n.n, n.sat);
                    if (cls >= 2) continue;
                    const uint64_t uo = (need_u[kk] && ucap[kk]) ? need_u[kk] : 0;
                    const int c = usw_of(kk, uo);
                    if (c >= 0) Lc[n.dir & 63][cls][c]++;
                    else if (need_full[kk] || need_u[kk]) F[n.dir & 63][cls]++;
                }
                uint32_t pick[64][2] = {{0}};                 // bit d: U_d candidates get their own packs
                for (uint32_t dd = 0; dd < kb->dirs.size() && dd < 64; ++dd)
                    for (int cls = 0; cls < 2; ++cls) {
                        double best = 1e300;
                        for (uint32_t sub = 0; sub < (1u << kMaxUDirs); ++sub) {
                            double cost = 0;
                            uint32_t joined = F[dd][cls];
                            for (uint32_t d = 0; d < kMaxUDirs; ++d) {
                                if (!Lc[dd][cls][d]) continue;
                                if (sub >> d & 1) cost += ((Lc[dd][cls][d] + 255) / 256) * (0.20 + 1.22 * kb->dirs[dd].usw[d].frac);
                                else joined += Lc[dd][cls][d];
                            }
                            cost += ((joined + 255) / 256) * 1.42;
                            if (cost < best - 1e-9) { best = cost; pick[dd][cls] = sub; }
                        }
                    }
                for (uint32_t kk = lo; kk < hi; ++kk) {
                    const CNode &n = p->nodes[list[kk]];
                    if (n.kind != NK_RESTRICT) continue;
                    const uint32_t cls = slice_class(n.pred, n.n, n.sat);
                    if (cls >= 2) continue;
                    const uint64_t uo = (need_u[kk] && ucap[kk]) ? need_u[kk] : 0;
                    const int c = usw_of(kk, uo);
                    if (c >= 0 && (pick[n.dir & 63][cls] >> c & 1)) uswd[kk] = (int8_t)c;
                }
            }
            for (uint32_t kk = lo; kk < hi; ++kk) {
                const CNode &n = p->nodes[list[kk]];
                if (n.kind != NK_RESTRICT) continue;
                if (need_u[kk] && !ucap[kk]) need_full[kk] = 1;
                const uint64_t uo = (need_u[kk] && ucap[kk]) ? need_u[kk] : 0;
                const bool swept = uswd[kk] >= 0;             // U sweeps are always packed, separately
                if ((need_full[kk] || (uo && !swept)) && slice_class(n.pred, n.n, n.sat) < 2) nfull_dir[n.dir & 63]++;
                if (uo && !swept) uforce |= 1ull << (n.dir & 63);
            }
            par_for(hi - lo, 1 << 13, [&](size_t a, size_t b) {
                for (size_t kk = lo + a; kk < lo + b; ++kk) {
                    const CNode &n = p->nodes[list[kk]];
                    const bool isbool = n.kind == NK_AND || n.kind == NK_OR;
                    const uint64_t nu = need_u[kk];
                    uint64_t uo = 0;
                    if (nu) {
                        if (ucap[kk]) uo = nu;
                        else need_full[kk] = by_pack[kk] = 1;   // the EX packs read its full row
                    }
                    u_out[kk] = uo;
                    pmode[kk] = isbool && !need_full[kk] && (need_proj[kk] || cover_of_node[kk] >= 0);
                    const bool ex = use_u && n.kind == NK_RESTRICT && !need_full[kk] && !uo &&
                                    slice_class(n.pred, n.n, n.sat) < 2;
                    // a full-row restriction that runs in a lane pack (else: the per-node kernel)
                    const bool packed = n.kind == NK_RESTRICT && (need_full[kk] || uo) && use_slice &&
                                        slice_class(n.pred, n.n, n.sat) < 2 &&
                                        (uswd[kk] >= 0 || slice_worthwhile(kb, nfull_dir[n.dir & 63], force_slice) ||
                                         (uforce >> (n.dir & 63) & 1));
                    // a boolean only lane packs read in full: fused into those packs, no row
                    const bool fuse = allow_fuse && isbool && need_full[kk] && by_pack[kk] && !by_other[kk] && !need_proj[kk] &&
                                      cover_of_node[kk] < 0 && n.op_count >= 1 && n.op_count <= kFuseMaxOps;
                    fused[kk] = fuse;
                    for (uint32_t q = 0; q < n.op_count; ++q) {
                        const uint32_t o = p->ops[n.op_begin + q];
                        if (ref_type(o) != RT_NODE) continue;
                        const uint32_t lo2 = local[ref_id(o)];
                        if (ex) {
                            __atomic_fetch_or(&need_u[lo2], 1ull << n.dir, __ATOMIC_RELAXED);
                        } else if (!isbool) {
                            need_full[lo2] = 1;
                            if (packed) by_pack[lo2] = 1;
                            else by_other[lo2] = 1;
                        } else {
                            if (need_full[kk]) need_full[lo2] = by_other[lo2] = 1;
                            if (pmode[kk]) need_proj[lo2] = 1;
                            if (uo) __atomic_fetch_or(&need_u[lo2], uo, __ATOMIC_RELAXED);
                        }
                    }
                }
            });
            hi = lo;
        }
        // fused booleans have no row of their own (their operands' rows were demanded above)
        par_for(nn, 1 << 15, [&](size_t a, size_t b) {
            for (size_t k = a; k < b; ++k)
                if (fused[k]) need_full[k] = 0;
        });
        const double ts1 = now_ms();
        slot.assign(nn, 0);
        pslot.assign(nn, 0);
        const uint32_t nrows = par_rank(nn, [&](size_t k) { return need_full[k] != 0; }, slot);
        const uint32_t nprows = par_rank(nn, [&](size_t k) { return need_proj[k] != 0; }, pslot);
        cp.nrows = nrows;
        cp.nprows = nprows;
        // U-row slots: one per direction a boolean computes a U row for
        auto &ubase = tmp.ubase;
        ubase.assign(nn, 0);
        uint32_t nurows = 0;
        for (int pass = 0; pass < 2; ++pass) {      // restrictions' U rows first: zeroed per chunk
            for (uint32_t k = 0; k < nn; ++k) {
                if ((p->nodes[list[k]].kind == NK_RESTRICT) != (pass == 0)) continue;
                ubase[k] = nurows;
                nurows += (uint32_t)__builtin_popcountll(u_out[k]);
            }
            if (pass == 0) cp.nurows_r = nurows;
        }
        cp.nurows = nurows;
        // launch groups: (level, kind, dir) runs of the list; boolean runs split by full/projected
        groups.clear();
        members.clear();
        members.reserve(nn);
        for (uint32_t k = 0; k < nn;) {
            const CNode &a = p->nodes[list[k]];
            const uint8_t kind = (a.kind == NK_OR) ? NK_AND : a.kind;   // AND and OR share a launch
            const uint16_t key = (kind == NK_AND) ? 0 : a.dir;
            uint32_t e = k + 1;
            while (e < nn) {
                const CNode &b = p->nodes[list[e]];
                const uint8_t kb2 = (b.kind == NK_OR) ? NK_AND : b.kind;
                if (b.level != a.level || kb2 != kind || (kind != NK_AND && b.dir != key)) break;
                ++e;
            }
            if (kind == NK_AND) {
                for (int pm = 0; pm < 2; ++pm) {               // full rows, example-projected rows
                    Group g{kind, key, (uint32_t)members.size(), 0};
                    g.proj = pm;
                    for (uint32_t q = k; q < e; ++q)
                        if (pm ? pmode[q] != 0 : need_full[q] != 0) members.push_back(q);
                    g.count = (uint32_t)members.size() - g.first;
                    if (g.count) groups.push_back(g);
                }
                uint64_t dirs_u = 0;                           // then one group per U direction
                for (uint32_t q = k; q < e; ++q) dirs_u |= u_out[q];
                for (; dirs_u; dirs_u &= dirs_u - 1) {
                    const int d = __builtin_ctzll(dirs_u);
                    Group g{kind, key, (uint32_t)members.size(), 0};
                    g.usp = (int16_t)d;
                    for (uint32_t q = k; q < e; ++q)
                        if (u_out[q] >> d & 1) members.push_back(q);
                    g.count = (uint32_t)members.size() - g.first;
                    groups.push_back(g);
                }
            } else if (kind == NK_RESTRICT && use_slice) {
                // lane-packable nodes (class 0/1 sort first) needed in full -- packed when there
                // are enough of them -- then those needed only at the examples (EX packs over U
                // rows, always packed), then the per-node rest
                uint32_t ns = 0, nf = 0;
                bool any_u = false;
                auto in_full = [&](uint32_t q) { return need_full[q] || (u_out[q] && tmp.uswd[q] < 0); };
                while (k + ns < e && slice_class(p->nodes[list[k + ns]].pred, p->nodes[list[k + ns]].n,
                                                 p->nodes[list[k + ns]].sat) != 2) {
                    const uint32_t q = k + ns;
                    nf += in_full(q);
                    any_u |= u_out[q] && tmp.uswd[q] < 0;
                    ++ns;
                }
                const bool full_packs = nf && (slice_worthwhile(kb, nf, force_slice) || any_u);
                const uint32_t first_rest = (uint32_t)members.size();
                if (full_packs) {
                    Group g{kind, key, (uint32_t)members.size(), 0};
                    g.slice = true;
                    for (uint32_t q = k; q < k + ns; ++q)
                        if (in_full(q)) members.push_back(q);
                    g.count = (uint32_t)members.size() - g.first;
                    groups.push_back(g);
                }
                for (int d = 0; d < (int)kMaxUDirs; ++d) {     // U sweeps, one group per U direction
                    Group g{kind, key, (uint32_t)members.size(), 0};
                    g.slice = true;
                    g.usw = (int8_t)d;
                    for (uint32_t q = k; q < k + ns; ++q)
                        if (!need_full[q] && u_out[q] && tmp.uswd[q] == d) members.push_back(q);
                    g.count = (uint32_t)members.size() - g.first;
                    if (g.count) groups.push_back(g);
                }
                // EX packs: fillers available as U rows of this direction (U-space booleans,
                // atoms, TOP) in one group, fillers with full rows in another
                auto u_filler = [&](uint32_t q) {
                    const uint32_t c = p->ops[p->nodes[list[q]].op_begin];
                    return use_u && (ref_type(c) != RT_NODE || (u_out[local[ref_id(c)]] >> key & 1));
                };
                for (int uc = 1; uc >= 0 && ns > nf; --uc) {      // (nf counts the full-pack members)
                    Group g{kind, key, (uint32_t)members.size(), 0};
                    g.slice = true;
                    g.ex = true;
                    g.ucomp = uc;
                    for (uint32_t q = k; q < k + ns; ++q)
                        if (!need_full[q] && !u_out[q] && u_filler(q) == (bool)uc) members.push_back(q);
                    g.count = (uint32_t)members.size() - g.first;
                    if (g.count) groups.push_back(g);
                }
                (void)first_rest;
                Group g{kind, key, (uint32_t)members.size(), 0};
                if (!full_packs)
                    for (uint32_t q = k; q < k + ns; ++q)
                        if (need_full[q]) members.push_back(q);
                for (uint32_t q = k + ns; q < e; ++q) members.push_back(q);
                g.count = (uint32_t)members.size() - g.first;
                if (g.count) groups.push_back(g);
            } else if (kind == NK_DRANGE) {
                // ranges needed in full / projected / as roots, then one group per U direction
                Group g{kind, key, (uint32_t)members.size(), 0};
                for (uint32_t q = k; q < e; ++q)
                    if (need_full[q] || need_proj[q] || cover_of_node[q] >= 0 || !u_out[q]) members.push_back(q);
                g.count = (uint32_t)members.size() - g.first;
                if (g.count) groups.push_back(g);
                uint64_t dirs_u = 0;
                for (uint32_t q = k; q < e; ++q) dirs_u |= u_out[q];
                for (; dirs_u; dirs_u &= dirs_u - 1) {
                    const int d = __builtin_ctzll(dirs_u);
                    Group gu{kind, key, (uint32_t)members.size(), 0};
                    gu.usp = (int16_t)d;
                    for (uint32_t q = k; q < e; ++q)
                        if (u_out[q] >> d & 1) members.push_back(q);
                    gu.count = (uint32_t)members.size() - gu.first;
                    groups.push_back(gu);
                }
            } else {
                const uint32_t first = (uint32_t)members.size();
                for (uint32_t q = k; q < e; ++q) members.push_back(q);
                groups.push_back(Group{kind, key, first, e - k});
            }
            k = e;
        }
        // descriptor bases per group and operand bases per boolean member (for the parallel fill)
        size_t n_ops = 0, n_bool = 0, n_res = 0, n_dr = 0, n_str = 0;
        tmp.gdesc.resize(groups.size());
        tmp.opbase.assign(members.size(), 0);
        for (size_t gi = 0; gi < groups.size(); ++gi) {
            const Group &g = groups[gi];
            if (g.kind == NK_AND) {
                tmp.gdesc[gi] = (uint32_t)n_bool;
                n_bool += g.count;
                for (uint32_t m = g.first; m < g.first + g.count; ++m) {
                    tmp.opbase[m] = (uint32_t)n_ops;
                    n_ops += p->nodes[list[members[m]]].op_count;
                }
            } else if (g.kind == NK_RESTRICT) {
                tmp.gdesc[gi] = (uint32_t)n_res;
                n_res += g.count;
                if (!g.slice) *heavy_need = std::max(*heavy_need, restrict_scratch_bytes(kb, g.key, g.count));
                if (g.slice && !g.ucomp)            // fused fillers: their operands, read by the pack
                    for (uint32_t m = g.first; m < g.first + g.count; ++m) {
                        const uint32_t c = p->ops[p->nodes[list[members[m]]].op_begin];
                        if (ref_type(c) != RT_NODE || !tmp.fused[local[ref_id(c)]]) continue;
                        tmp.opbase[m] = (uint32_t)n_ops;
                        n_ops += p->nodes[ref_id(c)].op_count;
                    }
            } else if (g.kind == NK_STRING) {
                tmp.gdesc[gi] = (uint32_t)n_str;
                n_str += g.count;
            } else {
                tmp.gdesc[gi] = (uint32_t)n_dr;
                n_dr += g.count;
            }
        }
        cp.off_bool = 0;
        cp.off_ops = align_up(cp.off_bool + n_bool * sizeof(BoolDesc), 16);
        cp.off_res = align_up(cp.off_ops + n_ops * sizeof(Operand), 16);
        cp.off_dr = align_up(cp.off_res + n_res * sizeof(RestrictDesc), 16);
        cp.off_str = align_up(cp.off_dr + n_dr * sizeof(DrangeDesc), 16);
        cp.off_cov = align_up(cp.off_str + n_str * sizeof(StringDesc), 16);
        cp.off_rows = align_up(cp.off_cov + nroots * sizeof(uint32_t), 16);
        cp.blob_bytes = align_up(cp.off_rows + (out_bits ? nroots * sizeof(void *) : 0), 256);
        cp.blob_off = *blob_cursor;
        *blob_cursor += cp.blob_bytes;
        timing_note("plan: covers+demands", ts1 - ts0);
        timing_note("plan: slots+groups", now_ms() - ts1);
        if (timing_enabled()) {            // plan statistics (HEDL_TIMING=1): lanes per pack kind
            uint64_t full_rows = 0, full_u_only = 0, full_any = 0, ex_u = 0, ex_full = 0, per_node = 0, fused_n = 0, swept = 0;
            uint64_t bool_full = 0, bool_proj = 0, bool_u = 0, restr_fillers_full = 0;
            for (const Group &g : groups)
                for (uint32_t m = g.first; m < g.first + g.count; ++m) {
                    const uint32_t q = members[m];
                    if (g.kind == NK_RESTRICT) {
                        if (g.usw >= 0) {
                            ++swept;
                        } else if (g.slice && !g.ex) {
                            ++full_any;
                            if (need_full[q]) ++full_rows; else ++full_u_only;
                        } else if (g.ex) { if (g.ucomp) ++ex_u; else ++ex_full; }
                        else ++per_node;
                    } else if (g.kind == NK_AND) {
                        if (g.usp >= 0) ++bool_u; else if (g.proj) ++bool_proj; else ++bool_full;
                    }
                }
            for (uint32_t k = 0; k < nn; ++k) {
                fused_n += tmp.fused[k];
                if (p->nodes[list[k]].kind == NK_RESTRICT && tmp.by_pack[k] && need_full[k]) ++restr_fillers_full;
            }
            if (std::getenv("HEDL_PLAN_GROUPS"))   // per full-pack group: level dir class lanes (U-only lanes by dir mask)
                for (const Group &g : groups) {
                    if (g.kind != NK_RESTRICT || !g.slice || g.ex) continue;
                    uint32_t byu[16] = {0}, nfr = 0;
                    const CNode &n0 = p->nodes[list[members[g.first]]];
                    for (uint32_t m = g.first; m < g.first + g.count; ++m) {
                        const uint32_t q = members[m];
                        if (need_full[q]) ++nfr; else byu[tmp.u_out[q] & 15]++;
                    }
                    std::fprintf(stderr, "[hedl group] level %u dir %u lanes %u full %u U-only by mask:", n0.level, g.key,
                                 g.count, nfr);
                    for (int b = 1; b < 16; ++b) if (byu[b]) std::fprintf(stderr, " %x:%u", b, byu[b]);
                    std::fprintf(stderr, "\n");
                }
            std::fprintf(stderr, "[hedl plan] U sweeps %llu\n", (unsigned long long)swept);
            std::fprintf(stderr, "[hedl plan] restrict: full-pack %llu (full row %llu, U rows only %llu), EX over U %llu, "
                                 "EX over full rows %llu, per-node %llu; bool: full %llu, projected %llu, U %llu, fused %llu; "
                                 "restrictions read in full by packs %llu\n",
                         (unsigned long long)full_any, (unsigned long long)full_rows, (unsigned long long)full_u_only,
                         (unsigned long long)ex_u, (unsigned long long)ex_full, (unsigned long long)per_node,
                         (unsigned long long)bool_full, (unsigned long long)bool_proj, (unsigned long long)bool_u,
                         (unsigned long long)fused_n, (unsigned long long)restr_fillers_full);
        }
        return;
    }

    char *h = h_blob + cp.blob_off;
    auto ptr_of = [&](uint32_t r) -> const uint32_t * {        // full row of an operand
        switch (ref_type(r)) {
        case RT_NODE: return rows + (size_t)slot[local[ref_id(r)]] * kb->W4;
        case RT_ATOM: return kb->concepts + (size_t)ref_id(r) * kb->W4;
        default: return kb->ones;
        }
    };
    auto pptr_of = [&](uint32_t r) -> const uint32_t * {       // projected row of an operand
        switch (ref_type(r)) {
        case RT_NODE: return prows + (size_t)pslot[local[ref_id(r)]] * kb->MW4;
        case RT_ATOM: return kb->pconcepts + (size_t)ref_id(r) * kb->MW4;
        default: return kb->pones;
        }
    };
    auto out_of = [&](uint32_t k) { return need_full[k] ? rows + (size_t)slot[k] * kb->W4 : nullptr; };
    // U rows: slot stride = the widest direction's UW4
    const auto &u_out = tmp.u_out;
    const auto &ubase = tmp.ubase;
    uint32_t uw4max = 0;
    for (const hedl_dir &x : kb->dirs) uw4max = std::max(uw4max, x.UW4);
    auto urow_of = [&](uint32_t k, int d) -> uint32_t * {
        return urows + (size_t)(ubase[k] + __builtin_popcountll(u_out[k] & ((1ull << d) - 1))) * uw4max;
    };
    auto uptr_of = [&](uint32_t r, int d) -> const uint32_t * {   // U row (direction d) of an operand
        switch (ref_type(r)) {
        case RT_NODE: return urow_of(local[ref_id(r)], d);
        case RT_ATOM: return kb->dirs[d].uconcepts + (size_t)ref_id(r) * kb->dirs[d].UW4;
        default: return kb->dirs[d].uones;
        }
    };
    auto proj_of = [&](uint32_t k) { return need_proj[k] ? prows + (size_t)pslot[k] * kb->MW4 : nullptr; };
    BoolDesc *hb = (BoolDesc *)(h + cp.off_bool);
    Operand *ho = (Operand *)(h + cp.off_ops);
    RestrictDesc *hr = (RestrictDesc *)(h + cp.off_res);
    DrangeDesc *hd = (DrangeDesc *)(h + cp.off_dr);
    StringDesc *hs = (StringDesc *)(h + cp.off_str);
    const Workspace *wsp = (const Workspace *)p->ws;
    // tasks: (group, member range); filled in parallel, each at precomputed offsets
    struct Task { uint32_t g, m0, m1; double bytes, bytes2; };
    std::vector<Task> tasks;
    for (uint32_t gi = 0; gi < groups.size(); ++gi)
        for (uint32_t m = groups[gi].first; m < groups[gi].first + groups[gi].count; m += 8192)
            tasks.push_back({gi, m, std::min(m + 8192, groups[gi].first + groups[gi].count), 0, 0});
    par_for(tasks.size(), nn < (1u << 15) ? tasks.size() : 1, [&](size_t t0, size_t t1) {
        for (size_t ti = t0; ti < t1; ++ti) {
            Task &T = tasks[ti];
            const Group &g = groups[T.g];
            const uint32_t base = tmp.gdesc[T.g];
            if (g.kind == NK_AND && g.usp >= 0) {             // evaluated over U of direction usp
                const double wb = 4.0 * kb->dirs[g.usp].UW;
                for (uint32_t m = T.m0; m < T.m1; ++m) {
                    const uint32_t k = members[m];
                    const CNode &n = p->nodes[list[k]];
                    BoolDesc bd;
                    bd.out = urow_of(k, g.usp);
                    bd.proj = nullptr;
                    uint32_t io = tmp.opbase[m];
                    bd.op_first = io;
                    bd.op_count = n.op_count;
                    bd.is_or = n.kind == NK_OR;
                    bd.cover = -1;
                    for (uint32_t q = 0; q < n.op_count; ++q) {
                        const uint32_t o = p->ops[n.op_begin + q];
                        ho[io++] = Operand{uptr_of(o, g.usp), ref_comp(o) ? 0xffffffffu : 0u, 0};
                    }
                    hb[base + (m - g.first)] = bd;
                    T.bytes += wb * (n.op_count + 1);
                }
            } else if (g.kind == NK_AND) {
                const double wb = 4.0 * (g.proj ? kb->MW : kb->W);
                for (uint32_t m = T.m0; m < T.m1; ++m) {
                    const uint32_t k = members[m];
                    const CNode &n = p->nodes[list[k]];
                    BoolDesc bd;
                    if (g.proj) {           // projected: the output (if any) is the projected row
                        bd.out = proj_of(k);
                        bd.proj = nullptr;
                    } else {
                        bd.out = out_of(k);
                        bd.proj = proj_of(k);
                    }
                    uint32_t io = tmp.opbase[m];
                    bd.op_first = io;
                    bd.op_count = n.op_count;
                    bd.is_or = n.kind == NK_OR;
                    bd.cover = cover_of_node[k];
                    for (uint32_t q = 0; q < n.op_count; ++q) {
                        const uint32_t o = p->ops[n.op_begin + q];
                        ho[io++] = Operand{g.proj ? pptr_of(o) : ptr_of(o), ref_comp(o) ? 0xffffffffu : 0u, 0};
                    }
                    hb[base + (m - g.first)] = bd;
                    T.bytes += wb * (n.op_count + (bd.out ? 1 : 0) + (bd.cover >= 0 ? 2 : 0));
                }
            } else if (g.kind == NK_RESTRICT) {
                const hedl_dir &dr = kb->dirs[g.key];
                for (uint32_t m = T.m0; m < T.m1; ++m) {
                    const uint32_t k = members[m];
                    const CNode &n = p->nodes[list[k]];
                    const uint32_t c = p->ops[n.op_begin];
                    RestrictDesc rd;
                    rd.op_first = rd.op_n = 0;
                    rd.uout = nullptr;
                    rd.udirs = rd.pad_ = 0;
                    if (u_out[k] && g.usw < 0) {             // full pack: U rows from the epilogue
                        rd.uout = urow_of(k, __builtin_ctzll(u_out[k]));
                        rd.udirs = (uint32_t)u_out[k];
                    }
                    if (!g.ucomp && ref_type(c) == RT_NODE && tmp.fused[local[ref_id(c)]]) {
                        // fused filler: the pack combines its operand rows (k-ary AND / OR with
                        // complement masks, Alg. 1-2) instead of reading a materialised row
                        const CNode &f = p->nodes[ref_id(c)];
                        uint32_t io = tmp.opbase[m];
                        rd.child = nullptr;
                        rd.op_first = io;
                        rd.op_n = f.op_count | (f.kind == NK_OR ? 0x80000000u : 0u);
                        for (uint32_t q = 0; q < f.op_count; ++q) {
                            const uint32_t o = p->ops[f.op_begin + q];
                            ho[io++] = Operand{ptr_of(o), ref_comp(o) ? 0xffffffffu : 0u, 0};
                        }
                    } else {
                        rd.child = g.ucomp ? uptr_of(c, g.key) : ptr_of(c);
                    }
                    rd.out = out_of(k);
                    rd.proj = proj_of(k);
                    rd.cmask = ref_comp(c) ? 0xffffffffu : 0u;
                    rd.pred = n.pred;
                    rd.n = n.n;
                    rd.sat = n.sat;
                    rd.cover = cover_of_node[k];
                    if (g.usw >= 0) rd.proj = urow_of(k, g.usw);   // U sweep: the U row is its output
                    rd.heavy_slot = (m - g.first) * dr.n_heavy;
                    hr[base + (m - g.first)] = rd;
                    T.bytes += 4.0 * (kb->N + 1) + 4.0 * (dr.E - dr.E_heavy) +
                               4.0 * kb->W * (1 + (rd.out ? 1 : 0) + (rd.cover >= 0 ? 2 : 0));
                    T.bytes2 += 4.0 * dr.E_heavy;
                }
            } else if (g.kind == NK_STRING) {
                for (uint32_t m = T.m0; m < T.m1; ++m) {
                    const uint32_t k = members[m];
                    const CNode &n = p->nodes[list[k]];
                    StringDesc sd;
                    sd.out = out_of(k);
                    sd.proj = proj_of(k);
                    sd.cover = cover_of_node[k];
                    sd.mode = n.pred;
                    sd.vid = n.pred == SM_EQUAL ? n.n : 0;
                    sd.pat = nullptr;
                    sd.pat_len = 0;
                    if (n.pred == SM_CONTAIN) {
                        sd.pat = wsp->pats + wsp->pat_off[n.n];
                        sd.pat_len = (uint32_t)(wsp->pat_off[n.n + 1] - wsp->pat_off[n.n]);
                    }
                    hs[base + (m - g.first)] = sd;
                    T.bytes += n.bytes - 4.0 * kb->W + 4.0 * kb->W * ((sd.out ? 1 : 0) + (sd.cover >= 0 ? 2 : 0));
                }
            } else {
                for (uint32_t m = T.m0; m < T.m1; ++m) {
                    const uint32_t k = members[m];
                    const CNode &n = p->nodes[list[k]];
                    DrangeDesc dd;
                    dd.lo = n.lo;
                    dd.hi = n.hi;
                    dd.prop = n.dir;
                    if (g.usp >= 0) {                    // evaluated at the members of U_usp
                        const hedl_dir &du = kb->dirs[g.usp];
                        dd.out = urow_of(k, g.usp);
                        dd.proj = nullptr;
                        dd.cover = -1;
                        T.bytes += 4.0 * du.n_u * 3 + 4.0 * du.UW;   // U list + two row pointers + values, U row
                    } else {
                        dd.out = out_of(k);
                        dd.proj = proj_of(k);
                        dd.cover = cover_of_node[k];
                        T.bytes += kb->data_bytes[n.dir] + 4.0 * kb->W * ((dd.out ? 1 : 0) + (dd.cover >= 0 ? 2 : 0));
                    }
                    hd[base + (m - g.first)] = dd;
                }
            }
        }
    });
    cp.recs.clear();
    for (uint32_t gi = 0; gi < groups.size(); ++gi) {
        const Group &g = groups[gi];
        LaunchRec lr{g.kind, g.key, g.slice, g.proj, g.ex, g.count, tmp.gdesc[gi], 0, 0};
        lr.usp = g.usp;
        lr.ucomp = g.ucomp;
        lr.usw = g.usw;
        cp.recs.push_back(lr);
    }
    for (const Task &T : tasks) {
        cp.recs[T.g].bytes += T.bytes;
        cp.recs[T.g].bytes2 += T.bytes2;
    }
    std::memcpy(h + cp.off_cov, cover_of_root.data(), nroots * sizeof(uint32_t));
    if (out_bits) {
        const uint32_t **hrows = (const uint32_t **)(h + cp.off_rows);
        for (uint32_t k = 0; k < nroots; ++k) hrows[k] = rows + (size_t)slot[local[p->root_node[cp.ri + k]]] * kb->W4;
    }
}

}  // namespace

namespace hedl {

// Phase D: the launches of one chunk.
hedl_status launch_chunk(const hedl_kb *kb, Workspace *w, const ChunkPlan &cp, uint32_t r0, uint32_t *out_bits,
                         hedl_counts *counts_dev, cudaStream_t s) {
    const KbDev kd{kb->N, kb->W, kb->W4, kb->pos, kb->neg, kb->ex_mask, kb->ex_base};
    const KbDev kp{kb->M, kb->MW, kb->MW4, kb->ppos, kb->pneg, nullptr, nullptr};   // example-projected space
    const char *d = (const char *)w->plan.dev + cp.blob_off;
    const char *h = (const char *)w->plan.host + cp.blob_off;
    hedl_counts *cov = (hedl_counts *)w->counts.p;
    const uint32_t nroots = cp.rc - cp.ri;
    launch_cover_init(s, cov, cp.ncov, kb->npos, kb->nneg);
    if (cp.nprows && kb->MW4)
        HEDL_CUDA(kb, cudaMemsetAsync(w->prows.p, 0, (size_t)cp.nprows * kb->MW4 * 4, s));   // scatter targets
    if (cp.nurows_r) {                                  // restrictions' U rows: atomicOr targets too
        uint32_t uw4max = 0;
        for (const hedl_dir &x : kb->dirs) uw4max = std::max(uw4max, x.UW4);
        HEDL_CUDA(kb, cudaMemsetAsync(w->urows.p, 0, (size_t)cp.nurows_r * uw4max * 4, s));
    }
    const bool tm = timing_enabled();
    double t_rec = tm ? now_ms() : 0.0;
    for (const LaunchRec &lr : cp.recs) {
        if (tm) {                                        // host time of the previous record's launches
            const double t = now_ms();
            if (t - t_rec > 1.0)
                std::fprintf(stderr, "[hedl timing] launch record %zu (kind %d, %u nodes) took %.3f ms of host time\n",
                             (size_t)(&lr - cp.recs.data()) - 1, (int)(&lr - 1)->kind, (&lr - 1)->count, t - t_rec);
            t_rec = t;
        }
        if (lr.kind == NK_AND) {
            KbDev kx = lr.proj ? kp : kd;
            if (lr.usp >= 0) {                                   // U space of one direction (no coverage)
                const hedl_dir &du = kb->dirs[lr.usp];
                kx = KbDev{du.n_u, du.UW, du.UW4, nullptr, nullptr, nullptr, nullptr};
            }
            launch_bool(s, kx, (const BoolDesc *)(d + cp.off_bool) + lr.first_desc, lr.count,
                        (const Operand *)(d + cp.off_ops), cov, lr.bytes, kb->npos, kb->nneg, !lr.proj && lr.usp < 0);

        } else if (lr.kind == NK_RESTRICT) {
            const hedl_dir &dr = kb->dirs[lr.key];
            const RestrictDesc *dd_desc = (const RestrictDesc *)(d + cp.off_res) + lr.first_desc;
            if (lr.slice) {
                hedl_status st = slice_run(kb, &w->slice.p, &w->slice.bytes, s, kd, lr.key,
                                           lr.cls >= 0 ? nullptr : (const RestrictDesc *)(h + cp.off_res) + lr.first_desc,
                                           dd_desc, lr.count, cov, lr.ex, lr.cls, lr.ucomp,
                                           (const Operand *)(d + cp.off_ops), lr.usw);
                if (st) return st;
            } else {
                DirDev dd{dr.row_ptr, dr.col, dr.heavy_x, dr.heavy_nchunks, dr.chunks, dr.n_heavy, dr.n_chunks,
                          dr.tiles, dr.order, dr.tile_slice, dr.sell_off, dr.sell_w, dr.sell_col, dr.n_tiles};
                if (restrict_push(kb, lr.count)) {       // direction-optimising (push) candidates
                    const hedl_dir &iv = kb->dirs[lr.key ^ 1];
                    DirDev di{iv.row_ptr, iv.col, iv.heavy_x, iv.heavy_nchunks, iv.chunks, iv.n_heavy, iv.n_chunks,
                              iv.tiles, iv.order, iv.tile_slice, iv.sell_off, iv.sell_w, iv.sell_col, iv.n_tiles};
                    uint32_t *push = (uint32_t *)((char *)w->heavy.p + restrict_heavy_bytes(kb, lr.key, lr.count));
                    launch_restrict(s, kd, dd, dd_desc, lr.count, cov, (uint32_t *)w->heavy.p, lr.bytes, lr.bytes2, &di,
                                    push, push_scratch_words(kb->N, kb->W4, true));
                } else {
                    launch_restrict(s, kd, dd, dd_desc, lr.count, cov, (uint32_t *)w->heavy.p, lr.bytes, lr.bytes2);
                }
            }
        } else if (lr.kind == NK_STRING) {
            const hedl_sdir &sdr = kb->sdirs[lr.key];
            launch_string(s, kd, StrDev{sdr.row_ptr, sdr.vid, sdr.dict_off, sdr.dict},
                          (const StringDesc *)(d + cp.off_str) + lr.first_desc, lr.count, cov, lr.bytes);
        } else {
            const hedl_data &dp = kb->data[lr.key];
            if (lr.usp >= 0) {
                const hedl_dir &du = kb->dirs[lr.usp];
                const KbDev ku{du.n_u, du.UW, du.UW4, nullptr, nullptr, nullptr, nullptr};
                launch_drange(s, ku, dp.row_ptr, dp.val, (const DrangeDesc *)(d + cp.off_dr) + lr.first_desc, lr.count,
                              cov, lr.bytes, du.ulist);
            } else {
                launch_drange(s, kd, dp.row_ptr, dp.val, (const DrangeDesc *)(d + cp.off_dr) + lr.first_desc, lr.count,
                              cov, lr.bytes);
            }
        }
    }
    launch_gather_counts(s, cov, (const uint32_t *)(d + cp.off_cov), counts_dev + (cp.ri - r0), nroots);
    if (out_bits)
        launch_gather_bits(s, (const uint32_t *const *)(d + cp.off_rows), out_bits + (size_t)(cp.ri - r0) * kb->W, kb->W,
                           nroots);
    HEDL_CUDA(kb, cudaGetLastError());
    return HEDL_OK;
}

}  // namespace hedl

namespace {

// Evaluate roots [r0, r1) of the program.  counts_dev: device hedl_counts[r1-r0];
// out_bits: device [r1-r0][W] or null.
// *counts_io == null: the counts go to the workspace's staging buffer (host-bound results),
// whose address is returned in *counts_io.
hedl_status run(const hedl_kb *kb, hedl_program *p, uint32_t r0, uint32_t r1, uint32_t *out_bits,
                hedl_counts **counts_io, cudaStream_t s, uint32_t eflags) {
    Workspace *w = ws_of(p);
    auto ensure_stage = [&]() -> hedl_status {
        if (*counts_io) return HEDL_OK;
        hedl_status st2 = grow(kb, s, w->stage, (size_t)(r1 - r0) * sizeof(hedl_counts), false, PR_COUNTS, w);
        if (!st2) *counts_io = (hedl_counts *)w->stage.p;
        return st2;
    };
    if (w->used && w->last_stream != s && w->done) HEDL_CUDA(kb, cudaStreamWaitEvent(s, w->done, 0));
    PlanCache &pc = w->plan;
    const bool bits = out_bits != nullptr;
    const bool hit = pc.valid && pc.r0 == r0 && pc.r1 == r1 && pc.bits == bits && pc.eflags == eflags &&
                     pc.rows_base == w->rows.p && pc.heavy_base == w->heavy.p && pc.prows_base == w->prows.p &&
                     pc.urows_base == w->urows.p;
    hedl_status st;
    if (!hit) {
        // the previous plan's blobs may still be read by queued work: wait, then reuse them
        if (w->used && w->done) HEDL_CUDA(kb, cudaEventSynchronize(w->done));
        invalidate_plan(pc);
        if (w->ext) {
            // caller's block: every buffer is re-carved from its start for the new plan (the
            // queued work reading the old carve finished above); the staging of host-bound
            // counts is always carved, so later calls of this range never need more
            w->ext_used = 0;
            for (DevBuf *b : {&w->rows, &w->prows, &w->heavy, &w->counts, &w->slice, &w->stage, &w->urows}) *b = DevBuf();
            pc.dev = nullptr;
            pc.cap = 0;
            w->pats = nullptr;
            if ((st = grow(kb, s, w->stage, (size_t)(r1 - r0) * sizeof(hedl_counts), false, PR_COUNTS, w))) return st;
        }
        const size_t row_bytes = (size_t)kb->W4 * 4;
        if (!p->ws_limit) {            // default: half the free device memory, at most 48 GiB
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            p->ws_limit = std::max<uint64_t>(1ull << 28, std::min<uint64_t>(fr / 2, 48ull << 30));
        }
        const uint64_t lim = w->ext ? std::min<uint64_t>(p->ws_limit, w->ext_bytes) : p->ws_limit;
        const uint64_t row_cap = std::max<uint64_t>(1, row_bytes ? lim / row_bytes : (1ull << 22));
        if (!p->patterns.empty() && !w->pats) {      // the program's CONTAIN patterns, uploaded once
            std::vector<uint8_t> blob;
            w->pat_off.assign(1, 0);
            for (const std::string &q : p->patterns) {
                blob.insert(blob.end(), q.begin(), q.end());
                w->pat_off.push_back(blob.size());
            }
            if (w->ext) {
                if ((st = carve(kb, s, w, (void **)&w->pats, std::max<size_t>(blob.size(), 16), false))) return st;
            } else if (dev_malloc((void **)&w->pats, std::max<size_t>(blob.size(), 16), s) != cudaSuccess) {
                cudaGetLastError();
                w->pats = nullptr;
                return fail(HEDL_ERR_OOM, "pattern table");
            }
            HEDL_CUDA(kb, cudaMemcpy(w->pats, blob.data(), blob.size(), cudaMemcpyHostToDevice));
            count_io(blob.size(), 0);
        }
        const bool use_slice = !(eflags & HEDL_EVAL_PER_NODE) && slice_enabled(kb);
        const bool force = eflags & HEDL_EVAL_FORCE_SLICE;
        std::vector<std::vector<uint32_t>> lists;
        std::vector<std::pair<uint32_t, uint32_t>> ranges;
        const double t0 = now_ms();
        collect_chunks(p, r0, r1, row_cap, lists, ranges);
        const double t1 = now_ms();
        // phase B: sizes of every chunk, then the buffers (pointers become final)
        std::vector<uint32_t> local(p->nodes.size());
        pc.chunks.resize(lists.size());
        std::vector<ChunkTmp> tmps(lists.size());
        size_t cursor = 0, heavy_need = 16, max_nn = 1, max_cov = 1, max_np = 1, max_nu = 1;
        for (size_t c = 0; c < lists.size(); ++c) {
            ChunkPlan &cp = pc.chunks[c];
            cp.ri = ranges[c].first;
            cp.rc = ranges[c].second;
            fill_chunk(kb, p, lists[c], cp, bits, use_slice, force, !(eflags & HEDL_EVAL_NO_FUSE),
                       !(eflags & HEDL_EVAL_NO_RESTRICT_U), !(eflags & HEDL_EVAL_NO_USWEEP), nullptr, nullptr, nullptr,
                       local, nullptr, &cursor,
                       &heavy_need, true, tmps[c]);
            max_nn = std::max<size_t>(max_nn, cp.nrows);
            max_np = std::max<size_t>(max_np, cp.nprows);
            max_nu = std::max<size_t>(max_nu, cp.nurows);
            max_cov = std::max<size_t>(max_cov, cp.ncov);
        }
        const double tb = now_ms();
        if ((st = grow(kb, s, w->rows, max_nn * row_bytes + 16, false, PR_ROWS, w))) return st;
        if ((st = grow(kb, s, w->prows, max_np * kb->MW4 * 4 + 16, false, PR_PROWS, w))) return st;
        uint32_t uw4max = 0;
        for (const hedl_dir &x : kb->dirs) uw4max = std::max(uw4max, x.UW4);
        if ((st = grow(kb, s, w->urows, max_nu * uw4max * 4 + 16, false, PR_UROWS, w))) return st;
        if ((st = grow(kb, s, w->heavy, heavy_need, true, PR_HEAVY, w))) return st;
        if ((st = grow(kb, s, w->counts, max_cov * sizeof(hedl_counts), false, PR_COUNTS, w))) return st;
        if ((st = reserve_plan(kb, pc, std::max<size_t>(cursor, 256), w))) return st;
        bool any_slice = false;
        for (const ChunkTmp &t : tmps)
            for (const Group &g : t.groups) any_slice |= g.slice;
        // lane-pack scratch: allocated lazily by slice_run, carved here in caller-workspace mode
        if (w->ext && any_slice && (st = grow(kb, s, w->slice, slice_ws_bytes(kb), true, PR_SLICE, w))) return st;
        if ((st = ensure_stage())) return st;
        const double t2 = now_ms();
        timing_note("plan: buffers", t2 - tb);
        pc.r0 = r0; pc.r1 = r1; pc.bits = bits; pc.eflags = eflags;
        pc.rows_base = w->rows.p;
        pc.heavy_base = w->heavy.p;
        pc.prows_base = w->prows.p;
        pc.urows_base = w->urows.p;
        // phase C + D interleaved: fill chunk c on the host while chunk c-1 runs on the GPU
        for (size_t c = 0; c < lists.size(); ++c) {
            ChunkPlan &cp = pc.chunks[c];
            size_t cur = cp.blob_off;
            fill_chunk(kb, p, lists[c], cp, bits, use_slice, force, !(eflags & HEDL_EVAL_NO_FUSE),
                       !(eflags & HEDL_EVAL_NO_RESTRICT_U), !(eflags & HEDL_EVAL_NO_USWEEP), (uint32_t *)w->rows.p,
                       (uint32_t *)w->prows.p,
                       (uint32_t *)w->urows.p, local, (char *)pc.host, &cur, &heavy_need, false, tmps[c]);
            tmps[c] = ChunkTmp();   // release the chunk's planning state
            timing_note("plan: fill chunk", now_ms() - t2);
            HEDL_CUDA(kb, cudaMemcpyAsync((char *)pc.dev + cp.blob_off, (char *)pc.host + cp.blob_off, cp.blob_bytes,
                                          cudaMemcpyHostToDevice, s));
            count_io(cp.blob_bytes, 0);
            if ((st = launch_chunk(kb, w, cp, r0, out_bits, *counts_io, s))) { invalidate_plan(pc); return st; }
        }
        pc.valid = true;
        timing_note("plan: collect chunks", t1 - t0);
        timing_note("plan: sizes+buffers", t2 - t1);
        timing_note("plan: fill+upload+launch", now_ms() - t2);
    } else {
        if ((st = ensure_stage())) return st;
        if ((st = replay_plan(kb, w, r0, out_bits, *counts_io, s))) return st;
    }
    if (!w->done) HEDL_CUDA(kb, cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming));
    HEDL_CUDA(kb, cudaEventRecord(w->done, s));
    w->last_stream = s;
    w->used = true;
    return HEDL_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev); else prev = -1;
    }
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

}  // namespace

extern "C" hedl_status hedl_eval_batch(const hedl_kb *kb, hedl_program *p, uint32_t first, uint32_t n,
                                       uint32_t *out_bits, hedl_counts *counts, void *stream, uint32_t flags) {
    if (!kb || !p || (n && !counts)) return fail(HEDL_ERR_INVALID_ARG, "null kb/program/counts");
    if (p->kb != kb) return fail(HEDL_ERR_INVALID_ARG, "program was compiled for another KB");
    if (kb->poisoned) return fail(HEDL_ERR_CUDA, "KB handle is poisoned by an earlier CUDA error");
    if ((uint64_t)first + n > prog_n_roots(p)) return fail(HEDL_ERR_OUT_OF_RANGE, "root range out of range");
    if (!n) return HEDL_OK;
    std::lock_guard<std::mutex> lk(p->mu);
    DeviceGuard dg(kb->device);
    cudaStream_t s = (cudaStream_t)stream;
    const bool host_out = !(flags & HEDL_EVAL_COUNTS_DEVICE);
    hedl_counts *dcounts = host_out ? nullptr : counts;    // null: the workspace's device staging
    Workspace *w = ws_of(p);
    const size_t cbytes = (size_t)n * sizeof(hedl_counts);
    if (host_out) {
        if (w->stage_host_n < n && n <= (1u << 16)) {  // small results go through pinned memory
            if (w->stage_host) cudaFreeHost(w->stage_host);
            w->stage_host = nullptr;
            w->stage_host_n = 0;
            if (cudaMallocHost((void **)&w->stage_host, std::max<size_t>(cbytes, 4096)) == cudaSuccess)
                w->stage_host_n = std::max<size_t>(cbytes, 4096) / sizeof(hedl_counts);
            else
                cudaGetLastError();
        }
    }
    const uint32_t ef = flags & ~HEDL_EVAL_COUNTS_DEVICE;
    hedl_status st;
    if (p->dev && !p->dev_downloaded) {
        // device-compiled program: plan on the device; a batch that needs several chunks
        // goes to the host planner (one download of the program)
        if (host_out) {
            if ((st = grow(kb, s, w->stage, cbytes, false, PR_COUNTS))) return st;
            dcounts = (hedl_counts *)w->stage.p;
        }
        st = dplan_run(kb, p, first, first + n, out_bits, dcounts, s, ef);
        if (st == HEDL_ERR_UNSUPPORTED && !(st = dc_download(p))) st = run(kb, p, first, first + n, out_bits, &dcounts, s, ef);
    } else {
        st = run(kb, p, first, first + n, out_bits, &dcounts, s, ef);
    }
    if (host_out && st == HEDL_OK) {
        const bool pinned = w->stage_host && w->stage_host_n >= n;
        cudaError_t e = cudaMemcpyAsync(pinned ? (void *)w->stage_host : (void *)counts, dcounts, cbytes,
                                        cudaMemcpyDeviceToHost, s);
        count_io(0, cbytes);
        if (e != cudaSuccess) return cuda_fail(kb, e, "count D2H");
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(kb, e, "eval_batch sync");
        if (pinned) std::memcpy(counts, w->stage_host, cbytes);
    }
    return st;
}

// Latency path: the root's sub-DAG (post-order, root last) as one interpreter launch
// when it fits (<= kInterpMaxNodes nodes, rows in shared memory); else the batch path.
static bool build_interp(const hedl_kb *kb, const hedl_program *p, uint32_t root_node, InterpProg &prog) {
    std::vector<uint32_t> order, local_of;
    std::vector<std::pair<uint32_t, uint32_t>> st;
    std::vector<uint32_t> seen;
    auto is_seen = [&](uint32_t id) { return std::find(seen.begin(), seen.end(), id) != seen.end(); };
    st.push_back({root_node, 0});
    seen.push_back(root_node);
    while (!st.empty()) {
        auto &top = st.back();
        const CNode &n = p->nodes[top.first];
        if (n.kind == NK_STRING) return false;     // string restrictions run on the batch path
        if (top.second < n.op_count) {
            const uint32_t o = p->ops[n.op_begin + top.second++];
            if (ref_type(o) == RT_NODE && !is_seen(ref_id(o))) {
                if (seen.size() >= kInterpMaxNodes) return false;
                seen.push_back(ref_id(o));
                st.push_back({ref_id(o), 0});
            }
            continue;
        }
        order.push_back(top.first);
        st.pop_back();
    }
    if ((size_t)order.size() * kb->W4 * 4 > interp_smem_limit()) return false;
    prog.n_nodes = (uint32_t)order.size();
    prog.n_ops = 0;
    prog.npos = kb->npos;
    prog.nneg = kb->nneg;
    for (uint32_t i = 0; i < order.size(); ++i) {
        const CNode &n = p->nodes[order[i]];
        if (prog.n_ops + n.op_count > kInterpMaxOps) return false;
        InterpNode &d = prog.nodes[i];
        d.kind = n.kind; d.pred = n.pred; d.dir = n.dir; d.n = n.n; d.sat = n.sat; d.lo = n.lo; d.hi = n.hi;
        d.op_begin = prog.n_ops;
        d.op_count = n.op_count;
        for (uint32_t q = 0; q < n.op_count; ++q) {
            uint32_t o = p->ops[n.op_begin + q];
            if (ref_type(o) == RT_NODE) {
                const uint32_t li = (uint32_t)(std::find(order.begin(), order.end(), ref_id(o)) - order.begin());
                o = mkref(RT_NODE, li, ref_comp(o));
                if (n.kind == NK_RESTRICT) prog.nodes[li].kind |= 0x80;   // read at any individual
            }
            prog.ops[prog.n_ops++] = o;
        }
    }
    return true;
}

extern "C" hedl_status hedl_eval_one(const hedl_kb *kb, hedl_program *p, uint32_t root, uint32_t *out_bits,
                                     hedl_counts *out, void *stream) {
    if (!out) return fail(HEDL_ERR_INVALID_ARG, "null out");
    if (!kb || !p) return fail(HEDL_ERR_INVALID_ARG, "null kb/program");
    if (p->kb != kb) return fail(HEDL_ERR_INVALID_ARG, "program was compiled for another KB");
    if (kb->poisoned) return fail(HEDL_ERR_CUDA, "KB handle is poisoned by an earlier CUDA error");
    if (root >= prog_n_roots(p)) return fail(HEDL_ERR_OUT_OF_RANGE, "root out of range");
    static thread_local InterpProg prog;   // ~5 KB: keep it off the stack
    // a single CTA wins while launch/sync overheads dominate; above ~64k individuals the
    // multi-CTA per-node kernels are faster (measured, tools/opbench.py)
    static const bool no_interp = std::getenv("HEDL_NO_INTERP") != nullptr;
    if (p->dev && kb->N && kb->N <= kInterpMaxN && !no_interp) {   // the interpreter reads the host program
        std::lock_guard<std::mutex> lk(p->mu);
        hedl_status st = dc_download(p);
        if (st) return st;
    }
    if (kb->N && kb->N <= kInterpMaxN && !no_interp && build_interp(kb, p, p->root_node[root], prog)) {
        std::lock_guard<std::mutex> lk(p->mu);
        DeviceGuard dg(kb->device);
        hedl_kb *mkb = const_cast<hedl_kb *>(kb);
        {
            std::lock_guard<std::mutex> lk2(mkb->interp_mu);
            hedl_status st = interp_prepare(mkb);
            if (st) return st;
        }
        if (!p->lat_host) {
            // [0] the counts, [1].tp the completion sequence number the kernel writes after them
            if (cudaHostAlloc((void **)&p->lat_host, 2 * sizeof(hedl_counts), cudaHostAllocMapped) != cudaSuccess ||
                cudaHostGetDevicePointer((void **)&p->lat_dev, p->lat_host, 0) != cudaSuccess) {
                cudaGetLastError();
                p->lat_host = nullptr;
                return fail(HEDL_ERR_OOM, "mapped counts");
            }
        }
        cudaStream_t s = (cudaStream_t)stream;
        Workspace *w = ws_of(p);
        if (w->used && w->done) HEDL_CUDA(kb, cudaStreamWaitEvent(s, w->done, 0));
        // completion: the kernel writes the counts, then (system-scope fence) this call's sequence
        // number into mapped host memory; spinning on it returns ~µs earlier than a stream
        // synchronisation.  The stream is still queried now and then, so a failed launch
        // surfaces as an error; HEDL_LAT_SYNC=1 synchronises the stream instead (A/B).
        static const bool lat_sync = std::getenv("HEDL_LAT_SYNC") != nullptr;
        prog.seq = ++p->lat_seq;
        volatile uint64_t *flag = &p->lat_host[1].tp;
        hedl_status st = interp_launch(kb, prog, p->lat_dev, out_bits, s);
        if (st) return st;
        bool done = false;
        if (!lat_sync) {
            for (uint32_t spin = 1; !(done = (*flag == prog.seq)); ++spin)
                if (!(spin & 1023) && cudaStreamQuery(s) != cudaErrorNotReady) {
                    done = *flag == prog.seq;
                    break;
                }
        }
        if (!done) HEDL_CUDA(kb, cudaStreamSynchronize(s));
        const volatile hedl_counts *vc = p->lat_host;
        out->tp = vc->tp;
        out->fp = vc->fp;
        out->fn = vc->fn;
        out->tn = vc->tn;
        return HEDL_OK;
    }
    return hedl_eval_batch(kb, p, root, 1, out_bits, out, stream, HEDL_EVAL_PER_NODE);
}

extern "C" hedl_status hedl_program_free(hedl_program *p) {
    if (!p) return HEDL_OK;
    if (p->ws) {
        Workspace *w = (Workspace *)p->ws;
        DeviceGuard dg(p->kb->device);
        if (w->done) cudaEventSynchronize(w->done);
        if (w->ext) {                   // buffers carved from the caller's block: not ours
            if (w->plan.host) cudaFreeHost(w->plan.host);
        } else {
            const int roles[] = {PR_ROWS, PR_PROWS, PR_HEAVY, PR_COUNTS, PR_SLICE, PR_UROWS};
            int ri = 0;
            for (DevBuf *b : {&w->rows, &w->prows, &w->heavy, &w->counts, &w->slice, &w->urows})
                pool_give(p->kb, roles[ri++], b->p, b->bytes);
            pool_give(p->kb, PR_COUNTS, w->stage.p, w->stage.bytes);
            pool_give(p->kb, PR_PLAN_HOST, w->plan.host, w->plan.cap);
            pool_give(p->kb, PR_PLAN_DEV, w->plan.dev, w->plan.cap);
            if (w->pats) dev_free(w->pats);
        }
        if (w->stage_host) cudaFreeHost(w->stage_host);
        w->plan.host = w->plan.dev = nullptr;
        release_plan(w->plan);
        if (w->done) cudaEventDestroy(w->done);
        if (p->lat_host) cudaFreeHost(p->lat_host);
        delete w;
    } else if (p->lat_host) {
        cudaFreeHost(p->lat_host);
    }
    const hedl_kb *kb = p->kb;
    if (p->dev) {
        DeviceGuard dg(kb->device);
        dplan_free(p);
        dc_free_arrays(p);
    }
    delete p;
    kb_release(kb);
    return HEDL_OK;
}

// Device bytes one hedl_eval_batch(first, n) of a host-compiled program needs from a caller's
// workspace: the sizing pass of the planner (run(), phases A-B) without any launch.
extern "C" hedl_status hedl_program_workspace_bytes(const hedl_kb *kb, hedl_program *p, uint32_t first, uint32_t n,
                                                    int with_bits, uint32_t eflags, uint64_t *bytes) {
    if (!kb || !p || !bytes) return fail(HEDL_ERR_INVALID_ARG, "null kb/program/bytes");
    if (p->kb != kb) return fail(HEDL_ERR_INVALID_ARG, "program was compiled for another KB");
    if (p->dev && !p->dev_downloaded) return fail(HEDL_ERR_UNSUPPORTED, "device-compiled programs plan on the device (use hedl_compile)");
    if ((uint64_t)first + n > prog_n_roots(p)) return fail(HEDL_ERR_OUT_OF_RANGE, "root range out of range");
    std::lock_guard<std::mutex> lk(p->mu);
    DeviceGuard dg(kb->device);
    eflags &= ~HEDL_EVAL_COUNTS_DEVICE;
    size_t total = 0;
    auto add = [&](size_t b) { total += align_up(std::max<size_t>(b, 1), 256); };
    add((size_t)n * sizeof(hedl_counts));                                       // counts staging
    if (!p->patterns.empty()) {
        size_t pb = 0;
        for (const std::string &q : p->patterns) pb += q.size();
        add(std::max<size_t>(pb, 16));
    }
    if (n) {
        if (!p->ws_limit) {
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            p->ws_limit = std::max<uint64_t>(1ull << 28, std::min<uint64_t>(fr / 2, 48ull << 30));
        }
        const size_t row_bytes = (size_t)kb->W4 * 4;
        const uint64_t row_cap = std::max<uint64_t>(1, row_bytes ? p->ws_limit / row_bytes : (1ull << 22));
        const bool use_slice = !(eflags & HEDL_EVAL_PER_NODE) && slice_enabled(kb);
        std::vector<std::vector<uint32_t>> lists;
        std::vector<std::pair<uint32_t, uint32_t>> ranges;
        collect_chunks(p, first, first + n, row_cap, lists, ranges);
        std::vector<uint32_t> local(p->nodes.size());
        size_t cursor = 0, heavy_need = 16, max_nn = 1, max_cov = 1, max_np = 1, max_nu = 1;
        bool any_slice = false;
        for (size_t c = 0; c < lists.size(); ++c) {
            ChunkPlan cp;
            ChunkTmp tmp;
            cp.ri = ranges[c].first;
            cp.rc = ranges[c].second;
            fill_chunk(kb, p, lists[c], cp, with_bits != 0, use_slice, eflags & HEDL_EVAL_FORCE_SLICE,
                       !(eflags & HEDL_EVAL_NO_FUSE), !(eflags & HEDL_EVAL_NO_RESTRICT_U), !(eflags & HEDL_EVAL_NO_USWEEP), nullptr, nullptr,
                       nullptr, local, nullptr, &cursor, &heavy_need, true, tmp);
            max_nn = std::max<size_t>(max_nn, cp.nrows);
            max_np = std::max<size_t>(max_np, cp.nprows);
            max_nu = std::max<size_t>(max_nu, cp.nurows);
            max_cov = std::max<size_t>(max_cov, cp.ncov);
            for (const Group &g : tmp.groups) any_slice |= g.slice;
        }
        uint32_t uw4max = 0;
        for (const hedl_dir &x : kb->dirs) uw4max = std::max(uw4max, x.UW4);
        add(max_nn * row_bytes + 16);
        add(max_np * kb->MW4 * 4 + 16);
        add(max_nu * uw4max * 4 + 16);
        add(heavy_need);
        add(max_cov * sizeof(hedl_counts));
        add(std::max<size_t>(std::max<size_t>(cursor, 256), 4096));             // device plan blob
        if (any_slice) add(slice_ws_bytes(kb));
    }
    *bytes = total;
    return HEDL_OK;
}

// Caller-provided workspace: every later evaluation of `p` carves its device buffers out of
// [ptr, ptr + bytes) and never allocates device memory (OOM when the block is too small).
extern "C" hedl_status hedl_program_set_workspace(hedl_program *p, void *ptr, uint64_t bytes) {
    if (!p) return fail(HEDL_ERR_INVALID_ARG, "null program");
    if (ptr && bytes < 4096) return fail(HEDL_ERR_INVALID_ARG, "workspace smaller than 4 KiB");
    if (p->dev && !p->dev_downloaded && ptr)
        return fail(HEDL_ERR_UNSUPPORTED, "device-compiled programs plan on the device (use hedl_compile)");
    std::lock_guard<std::mutex> lk(p->mu);
    DeviceGuard dg(p->kb->device);
    Workspace *w = ws_of(p);
    if (w->done) cudaEventSynchronize(w->done);
    invalidate_plan(w->plan);
    if (w->ext) {                       // detach: carved buffers are not ours to free
        for (DevBuf *b : {&w->rows, &w->prows, &w->heavy, &w->counts, &w->slice, &w->stage, &w->urows}) *b = DevBuf();
        w->plan.dev = nullptr;
        w->plan.cap = 0;
        w->pats = nullptr;
    } else {                            // library-owned buffers go back to the KB's pool
        const int roles[] = {PR_ROWS, PR_PROWS, PR_HEAVY, PR_COUNTS, PR_SLICE, PR_UROWS, PR_COUNTS};
        int ri = 0;
        for (DevBuf *b : {&w->rows, &w->prows, &w->heavy, &w->counts, &w->slice, &w->urows, &w->stage}) {
            pool_give(p->kb, roles[ri++], b->p, b->bytes);
            *b = DevBuf();
        }
        if (w->plan.dev) pool_give(p->kb, PR_PLAN_DEV, w->plan.dev, w->plan.cap);
        if (w->plan.host) pool_give(p->kb, PR_PLAN_HOST, w->plan.host, w->plan.cap);
        w->plan.dev = w->plan.host = nullptr;
        w->plan.cap = w->plan.host_cap = 0;
        if (w->pats) dev_free(w->pats);
        w->pats = nullptr;
    }
    w->ext = (char *)ptr;
    w->ext_bytes = ptr ? bytes : 0;
    w->ext_used = 0;
    return HEDL_OK;
}

extern "C" hedl_status hedl_program_set_workspace_limit(hedl_program *p, uint64_t bytes) {
    if (!p || bytes < (1u << 20)) return fail(HEDL_ERR_INVALID_ARG, "null program or limit < 1 MiB");
    std::lock_guard<std::mutex> lk(p->mu);
    p->ws_limit = bytes;
    if (p->ws) {
        Workspace *w = (Workspace *)p->ws;
        if (w->done) cudaEventSynchronize(w->done);
        invalidate_plan(w->plan);
    }
    return HEDL_OK;
}

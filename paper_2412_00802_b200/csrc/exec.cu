// Executor: hedl_eval_one / hedl_eval_batch.
//
// A set of roots is planned as one or more chunks.  Per chunk the needed
// canonical nodes are collected, grouped by topological level and then by
// (kind, role direction / data property), and each group runs as ONE launch
// whose blockIdx.y walks the group's nodes (consecutive nodes of one direction
// re-hit the same CSR in L2).  Root nodes fuse the Alg. 15 coverage
// (PAPER.md:548-553).  One H2D copy of descriptors per chunk; counts come back
// with one D2H per call (the paper's single cudaMemcpyAsync).
#include <algorithm>

#include "internal.h"
#include "slice.h"

using namespace hedl;

namespace {

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

// per-program device/pinned buffers (kept in hedl_program via an opaque side table)
struct Workspace {
    DevBuf rows, heavy, desc, counts, slice;
    void *pinned[2] = {nullptr, nullptr};
    size_t pinned_bytes[2] = {0, 0};
    cudaEvent_t pinned_ev[2] = {nullptr, nullptr};
    int pin_idx = 0;
    cudaEvent_t done = nullptr;
    cudaStream_t last_stream = nullptr;
    bool used = false;
};

Workspace *ws_of(hedl_program *p) {
    if (!p->ws) p->ws = new Workspace();
    return (Workspace *)p->ws;
}

hedl_status grow(const hedl_kb *kb, cudaStream_t s, DevBuf &b, size_t need, bool zero) {
    if (b.bytes >= need) return HEDL_OK;
    HEDL_CUDA(kb, cudaStreamSynchronize(s));
    size_t sz = std::max(need, b.bytes * 3 / 2);
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    sz = (sz + 255) & ~size_t(255);
    cudaError_t e = cudaMalloc(&b.p, sz);
    if (e != cudaSuccess) {
        cudaGetLastError();
        e = cudaMalloc(&b.p, need);
        if (e != cudaSuccess) { cudaGetLastError(); return fail(HEDL_ERR_OOM, "workspace allocation failed"); }
        sz = need;
    }
    b.bytes = sz;
    if (zero) HEDL_CUDA(kb, cudaMemsetAsync(b.p, 0, sz, s));
    return HEDL_OK;
}

hedl_status get_pinned(Workspace *w, size_t need, void **out) {
    const int i = w->pin_idx;
    if (w->pinned_ev[i]) cudaEventSynchronize(w->pinned_ev[i]);
    if (w->pinned_bytes[i] < need) {
        if (w->pinned[i]) cudaFreeHost(w->pinned[i]);
        size_t sz = std::max(need, w->pinned_bytes[i] * 3 / 2);
        if (cudaMallocHost(&w->pinned[i], sz) != cudaSuccess) {
            w->pinned[i] = nullptr;
            w->pinned_bytes[i] = 0;
            cudaGetLastError();
            return fail(HEDL_ERR_OOM, "pinned allocation failed");
        }
        w->pinned_bytes[i] = sz;
    }
    *out = w->pinned[i];
    return HEDL_OK;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Group {          // one launch
    uint8_t kind;       // NK_*
    uint16_t key;       // dir or prop
    uint32_t first, count;   // into the chunk node list
    bool slice = false;
};

// Evaluate roots [r0, r1) of the program as consecutive chunks.
// counts_dev: device hedl_counts[r1-r0] output; out_bits: device [r1-r0][W] or null.
hedl_status run(const hedl_kb *kb, hedl_program *p, uint32_t r0, uint32_t r1, uint32_t *out_bits,
                hedl_counts *counts_dev, cudaStream_t s, uint32_t eflags) {
    Workspace *w = ws_of(p);
    if (w->used && w->last_stream != s && w->done) HEDL_CUDA(kb, cudaStreamWaitEvent(s, w->done, 0));
    const size_t row_bytes = (size_t)kb->W4 * 4;
    const KbDev kd{kb->N, kb->W, kb->W4, kb->pos, kb->neg};
    const uint64_t max_nodes = std::max<uint64_t>(1, row_bytes ? p->ws_limit / row_bytes : (1ull << 20));
    const uint64_t node_cap = std::min<uint64_t>(max_nodes, 1u << 20);
    const bool use_slice = !(eflags & HEDL_EVAL_PER_NODE) && slice_enabled(kb);

    if (p->stamp.size() < p->nodes.size()) p->stamp.assign(p->nodes.size(), 0);
    std::vector<uint32_t> list, st, slot_of_node_tmp;
    std::vector<uint32_t> cover_of_root;   // per root in chunk: cover slot
    std::vector<uint32_t> local;           // node id -> index in list (valid when stamped)
    if (local.size() < p->nodes.size()) local.resize(p->nodes.size());
    std::vector<int32_t> cover_of_node;

    uint32_t ri = r0;
    while (ri < r1) {
        // ---- collect the chunk's nodes (DFS from roots, stamp-deduplicated) ----
        const uint32_t gen = ++p->stamp_gen;
        list.clear();
        uint32_t rc = ri;
        for (; rc < r1; ++rc) {
            const size_t before = list.size();
            st.assign(1, p->root_node[rc]);
            if (p->stamp[p->root_node[rc]] == gen) continue;
            p->stamp[p->root_node[rc]] = gen;
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
                    }
                }
            }
            if (list.size() > node_cap && rc > ri) {    // this root overflows: defer it
                for (size_t k = before; k < list.size(); ++k) p->stamp[list[k]] = 0;
                list.resize(before);
                break;
            }
        }
        const uint32_t nroots = rc - ri;
        // ---- order: level, kind, direction ----
        std::sort(list.begin(), list.end(), [&](uint32_t a, uint32_t b) {
            const CNode &x = p->nodes[a], &y = p->nodes[b];
            if (x.level != y.level) return x.level < y.level;
            if (x.kind != y.kind) return x.kind < y.kind;
            if (x.dir != y.dir) return x.dir < y.dir;
            if (x.kind == NK_RESTRICT) {
                const uint32_t cx = slice_class(x.pred, x.n, x.sat), cy = slice_class(y.pred, y.n, y.sat);
                if (cx != cy) return cx < cy;
            }
            return a < b;
        });
        const uint32_t nn = (uint32_t)list.size();
        for (uint32_t k = 0; k < nn; ++k) local[list[k]] = k;
        // cover slots: one per distinct root node of the chunk
        cover_of_node.assign(nn, -1);
        cover_of_root.resize(nroots);
        uint32_t ncov = 0;
        for (uint32_t k = 0; k < nroots; ++k) {
            const uint32_t li = local[p->root_node[ri + k]];
            if (cover_of_node[li] < 0) cover_of_node[li] = (int32_t)ncov++;
            cover_of_root[k] = (uint32_t)cover_of_node[li];
        }
        // groups
        std::vector<Group> groups;
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
            Group g{kind, key, k, e - k};
            if (use_slice && kind == NK_RESTRICT) {
                uint32_t ns = 0;   // leading lane-packable nodes (class 0/1 sort first)
                while (ns < g.count) {
                    const CNode &c = p->nodes[list[k + ns]];
                    if (slice_class(c.pred, c.n, c.sat) == 2) break;
                    ++ns;
                }
                if (ns && slice_worthwhile(kb, ns, eflags & HEDL_EVAL_FORCE_SLICE)) {
                    if (ns < g.count) {            // split: packable prefix + per-node rest
                        Group g1{kind, key, k, ns};
                        g1.slice = true;
                        groups.push_back(g1);
                        g.first = k + ns;
                        g.count -= ns;
                    } else {
                        g.slice = true;
                    }
                }
            }
            groups.push_back(g);
            k = e;
        }
        // ---- sizes ----
        size_t n_ops = 0, n_bool = 0, n_res = 0, n_dr = 0, heavy_need = 0;
        for (const Group &g : groups) {
            if (g.kind == NK_AND) {
                n_bool += g.count;
                for (uint32_t k = g.first; k < g.first + g.count; ++k) n_ops += p->nodes[list[k]].op_count;
            } else if (g.kind == NK_RESTRICT) {
                n_res += g.count;
                heavy_need = std::max(heavy_need, (size_t)g.count * kb->dirs[g.key].n_heavy * 8);
            } else {
                n_dr += g.count;
            }
        }
        const size_t off_bool = 0;
        const size_t off_ops = align_up(off_bool + n_bool * sizeof(BoolDesc), 16);
        const size_t off_res = align_up(off_ops + n_ops * sizeof(Operand), 16);
        const size_t off_dr = align_up(off_res + n_res * sizeof(RestrictDesc), 16);
        const size_t off_cov = align_up(off_dr + n_dr * sizeof(DrangeDesc), 16);
        const size_t off_rows = align_up(off_cov + nroots * sizeof(uint32_t), 16);
        const size_t desc_bytes = align_up(off_rows + (out_bits ? nroots * sizeof(void *) : 0), 16);

        hedl_status stt;
        if ((stt = grow(kb, s, w->rows, std::max<size_t>(16, nn * row_bytes), false))) return stt;
        if ((stt = grow(kb, s, w->heavy, std::max<size_t>(16, heavy_need), true))) return stt;
        if ((stt = grow(kb, s, w->desc, desc_bytes, false))) return stt;
        if ((stt = grow(kb, s, w->counts, std::max<size_t>(32, ncov * sizeof(hedl_counts)), false))) return stt;
        void *hp = nullptr;
        if ((stt = get_pinned(w, desc_bytes, &hp))) return stt;
        char *h = (char *)hp;
        char *d = (char *)w->desc.p;
        uint32_t *rows = (uint32_t *)w->rows.p;
        hedl_counts *cov = (hedl_counts *)w->counts.p;
        auto ptr_of = [&](uint32_t r) -> const uint32_t * {
            switch (ref_type(r)) {
            case RT_NODE: return rows + (size_t)local[ref_id(r)] * kb->W4;
            case RT_ATOM: return kb->concepts + (size_t)ref_id(r) * kb->W4;
            default: return kb->ones;
            }
        };
        // ---- fill descriptors (host, pinned) ----
        BoolDesc *hb = (BoolDesc *)(h + off_bool);
        Operand *ho = (Operand *)(h + off_ops);
        RestrictDesc *hr = (RestrictDesc *)(h + off_res);
        DrangeDesc *hd = (DrangeDesc *)(h + off_dr);
        uint32_t ib = 0, io = 0, ir = 0, idr = 0;
        struct LaunchRec { const Group *g; uint32_t first_desc; double bytes, bytes2; };
        std::vector<LaunchRec> recs;
        for (const Group &g : groups) {
            LaunchRec lr{&g, 0, 0, 0};
            if (g.kind == NK_AND) {
                lr.first_desc = ib;
                for (uint32_t k = g.first; k < g.first + g.count; ++k) {
                    const CNode &n = p->nodes[list[k]];
                    BoolDesc bd;
                    bd.out = rows + (size_t)k * kb->W4;
                    bd.op_first = io;
                    bd.op_count = n.op_count;
                    bd.is_or = n.kind == NK_OR;
                    bd.cover = cover_of_node[k];
                    for (uint32_t q = 0; q < n.op_count; ++q) {
                        const uint32_t o = p->ops[n.op_begin + q];
                        ho[io++] = Operand{ptr_of(o), ref_comp(o) ? 0xffffffffu : 0u, 0};
                    }
                    hb[ib++] = bd;
                    lr.bytes += n.bytes + (bd.cover >= 0 ? 8.0 * kb->W : 0);
                }
            } else if (g.kind == NK_RESTRICT) {
                lr.first_desc = ir;
                const hedl_dir &dr = kb->dirs[g.key];
                for (uint32_t k = g.first; k < g.first + g.count; ++k) {
                    const CNode &n = p->nodes[list[k]];
                    const uint32_t c = p->ops[n.op_begin];
                    RestrictDesc rd;
                    rd.child = ptr_of(c);
                    rd.out = rows + (size_t)k * kb->W4;
                    rd.cmask = ref_comp(c) ? 0xffffffffu : 0u;
                    rd.pred = n.pred;
                    rd.n = n.n;
                    rd.sat = n.sat;
                    rd.cover = cover_of_node[k];
                    rd.heavy_slot = (k - g.first) * dr.n_heavy;
                    hr[ir++] = rd;
                    lr.bytes += 4.0 * (kb->N + 1) + 4.0 * (dr.E - dr.E_heavy) + 8.0 * kb->W + (rd.cover >= 0 ? 8.0 * kb->W : 0);
                    lr.bytes2 += 4.0 * dr.E_heavy;
                }
            } else {
                lr.first_desc = idr;
                for (uint32_t k = g.first; k < g.first + g.count; ++k) {
                    const CNode &n = p->nodes[list[k]];
                    DrangeDesc dd;
                    dd.out = rows + (size_t)k * kb->W4;
                    dd.lo = n.lo;
                    dd.hi = n.hi;
                    dd.cover = cover_of_node[k];
                    dd.prop = n.dir;
                    hd[idr++] = dd;
                    lr.bytes += n.bytes + (dd.cover >= 0 ? 8.0 * kb->W : 0);
                }
            }
            recs.push_back(lr);
        }
        std::memcpy(h + off_cov, cover_of_root.data(), nroots * sizeof(uint32_t));
        if (out_bits) {
            const uint32_t **hrows = (const uint32_t **)(h + off_rows);
            for (uint32_t k = 0; k < nroots; ++k) hrows[k] = rows + (size_t)local[p->root_node[ri + k]] * kb->W4;
        }
        HEDL_CUDA(kb, cudaMemcpyAsync(d, h, desc_bytes, cudaMemcpyHostToDevice, s));
        count_io(desc_bytes, 0);
        if (!w->pinned_ev[w->pin_idx]) HEDL_CUDA(kb, cudaEventCreateWithFlags(&w->pinned_ev[w->pin_idx], cudaEventDisableTiming));
        HEDL_CUDA(kb, cudaEventRecord(w->pinned_ev[w->pin_idx], s));
        w->pin_idx ^= 1;

        // ---- launches ----
        launch_cover_init(s, cov, ncov, kb->npos, kb->nneg);
        for (const LaunchRec &lr : recs) {
            const Group &g = *lr.g;
            if (g.kind == NK_AND) {
                launch_bool(s, kd, (const BoolDesc *)(d + off_bool) + lr.first_desc, g.count,
                            (const Operand *)(d + off_ops), cov, lr.bytes);
            } else if (g.kind == NK_RESTRICT) {
                const hedl_dir &dr = kb->dirs[g.key];
                DirDev dd{dr.row_ptr, dr.col, dr.heavy_x, dr.heavy_nchunks, dr.chunks, dr.n_heavy, dr.n_chunks};
                const RestrictDesc *dd_desc = (const RestrictDesc *)(d + off_res) + lr.first_desc;
                if (g.slice) {
                    stt = slice_run(kb, &w->slice.p, &w->slice.bytes, s, kd, g.key, hr + lr.first_desc, dd_desc,
                                    g.count, cov);
                    if (stt) return stt;
                } else {
                    launch_restrict(s, kd, dd, dd_desc, g.count, cov, (uint32_t *)w->heavy.p, lr.bytes, lr.bytes2);
                }
            } else {
                const hedl_data &dp = kb->data[g.key];
                launch_drange(s, kd, dp.row_ptr, dp.val, (const DrangeDesc *)(d + off_dr) + lr.first_desc, g.count,
                              cov, lr.bytes);
            }
        }
        launch_gather_counts(s, cov, (const uint32_t *)(d + off_cov), counts_dev + (ri - r0), nroots);
        if (out_bits)
            launch_gather_bits(s, (const uint32_t *const *)(d + off_rows), out_bits + (size_t)(ri - r0) * kb->W, kb->W, nroots);
        HEDL_CUDA(kb, cudaGetLastError());
        ri = rc;
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
    if ((uint64_t)first + n > p->root_node.size()) return fail(HEDL_ERR_OUT_OF_RANGE, "root range out of range");
    if (!n) return HEDL_OK;
    std::lock_guard<std::mutex> lk(p->mu);
    DeviceGuard dg(kb->device);
    cudaStream_t s = (cudaStream_t)stream;
    hedl_counts *dcounts = counts;
    DevBuf out_stage;
    if (!(flags & HEDL_EVAL_COUNTS_DEVICE)) {
        cudaError_t e = cudaMallocAsync(&out_stage.p, (size_t)n * sizeof(hedl_counts), s);
        if (e != cudaSuccess) { cudaGetLastError(); return fail(HEDL_ERR_OOM, "count staging allocation failed"); }
        dcounts = (hedl_counts *)out_stage.p;
    }
    hedl_status st = run(kb, p, first, first + n, out_bits, dcounts, s, flags);
    if (!(flags & HEDL_EVAL_COUNTS_DEVICE)) {
        if (st == HEDL_OK) {
            cudaError_t e = cudaMemcpyAsync(counts, dcounts, (size_t)n * sizeof(hedl_counts), cudaMemcpyDeviceToHost, s);
            count_io(0, (uint64_t)n * sizeof(hedl_counts));
            if (e != cudaSuccess) st = cuda_fail(kb, e, "count D2H");
        }
        cudaFreeAsync(out_stage.p, s);
        if (st == HEDL_OK) {
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) st = cuda_fail(kb, e, "eval_batch sync");
        }
    }
    return st;
}

extern "C" hedl_status hedl_eval_one(const hedl_kb *kb, hedl_program *p, uint32_t root, uint32_t *out_bits,
                                     hedl_counts *out, void *stream) {
    if (!out) return fail(HEDL_ERR_INVALID_ARG, "null out");
    return hedl_eval_batch(kb, p, root, 1, out_bits, out, stream, HEDL_EVAL_PER_NODE);
}

extern "C" hedl_status hedl_program_free(hedl_program *p) {
    if (!p) return HEDL_OK;
    if (p->ws) {
        Workspace *w = (Workspace *)p->ws;
        DeviceGuard dg(p->kb->device);
        if (w->done) cudaEventSynchronize(w->done);
        for (DevBuf *b : {&w->rows, &w->heavy, &w->desc, &w->counts, &w->slice})
            if (b->p) cudaFree(b->p);
        for (int i = 0; i < 2; ++i) {
            if (w->pinned[i]) cudaFreeHost(w->pinned[i]);
            if (w->pinned_ev[i]) cudaEventDestroy(w->pinned_ev[i]);
        }
        if (w->done) cudaEventDestroy(w->done);
        delete w;
    }
    delete p;
    return HEDL_OK;
}

extern "C" hedl_status hedl_program_set_workspace_limit(hedl_program *p, uint64_t bytes) {
    if (!p || bytes < (1u << 20)) return fail(HEDL_ERR_INVALID_ARG, "null program or limit < 1 MiB");
    p->ws_limit = bytes;
    return HEDL_OK;
}

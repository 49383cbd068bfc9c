// hedl_kb_load: host build of the device KB layout, then upload.
//
// Paper: concepts matrix transposed (rows = concepts), roles as
// 2-column (subj, obj) matrices with an offset table, numeric
// concrete roles as (subj, value), examples matrix
// (PAPER.md:541).  Here: bit-packed rows padded to 16 B, per role a deduped
// CSR + transposed CSR (inverse roles), heavy-row chunk lists,
// per data property a CSR of ascending non-NaN values, example bitsets.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <thread>

#include "internal.h"

using namespace hedl;

namespace {

template <class F>
void parallel_ranges(uint64_t n, F f) {
    unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    if (n < (1u << 16) || nt == 1) { f(0, n); return; }
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        uint64_t a = n * t / nt, b = n * (t + 1) / nt;
        th.emplace_back([=] { f(a, b); });
    }
    for (auto &x : th) x.join();
}

struct HostCSR {
    std::vector<uint32_t> row_ptr, col;
};

// counting sort of (s, o) pairs by s, then sort + dedupe each row (sets)
// (objects < n_obj; n_obj = N for roles, the number of interned values for string roles)
hedl_status build_forward(uint32_t N, const uint32_t *s, const uint32_t *o, uint64_t m, HostCSR &out,
                          uint64_t n_obj = ~0ull) {
    if (n_obj == ~0ull) n_obj = N;
    std::vector<uint64_t> cnt(N + 1, 0);
    for (uint64_t k = 0; k < m; ++k) {
        if (s[k] >= N || o[k] >= n_obj) return fail(HEDL_ERR_OUT_OF_RANGE, "role assertion id >= N at index " + std::to_string(k));
        cnt[s[k] + 1]++;
    }
    for (uint32_t i = 0; i < N; ++i) cnt[i + 1] += cnt[i];
    std::vector<uint32_t> tmp(m);
    {
        std::vector<uint64_t> pos(cnt.begin(), cnt.end() - 1);
        for (uint64_t k = 0; k < m; ++k) tmp[pos[s[k]]++] = o[k];
    }
    std::vector<uint32_t> ucnt(N, 0);
    parallel_ranges(N, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) {
            auto first = tmp.begin() + cnt[i], last = tmp.begin() + cnt[i + 1];
            std::sort(first, last);
            ucnt[i] = (uint32_t)(std::unique(first, last) - first);
        }
    });
    out.row_ptr.assign(N + 1, 0);
    uint64_t acc = 0;
    for (uint32_t i = 0; i < N; ++i) {
        out.row_ptr[i] = (uint32_t)acc;
        acc += ucnt[i];
        if (acc > 0xffffffffull) return fail(HEDL_ERR_INVALID_ARG, "a role has >= 2^32 distinct assertions");
    }
    out.row_ptr[N] = (uint32_t)acc;
    out.col.resize(acc);
    parallel_ranges(N, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i)
            std::copy(tmp.begin() + cnt[i], tmp.begin() + cnt[i] + ucnt[i], out.col.begin() + out.row_ptr[i]);
    });
    return HEDL_OK;
}

// transposed CSR of a deduped CSR: rows = objects, sorted subjects (PAPER.md:299 swap)
void build_transpose(uint32_t N, const HostCSR &f, HostCSR &t) {
    t.row_ptr.assign(N + 1, 0);
    for (uint32_t y : f.col) t.row_ptr[y + 1]++;
    for (uint32_t i = 0; i < N; ++i) t.row_ptr[i + 1] += t.row_ptr[i];
    t.col.resize(f.col.size());
    std::vector<uint32_t> pos(t.row_ptr.begin(), t.row_ptr.end() - 1);
    for (uint32_t x = 0; x < N; ++x)
        for (uint32_t e = f.row_ptr[x]; e < f.row_ptr[x + 1]; ++e) t.col[pos[f.col[e]]++] = x;
}

template <class T>
hedl_status upload(hedl_kb *kb, cudaStream_t st, T **dst, const T *src, size_t n) {
    size_t bytes = std::max<size_t>(n * sizeof(T), 16);
    void *p = nullptr;
    cudaError_t e = dev_malloc(&p, bytes, st);
    if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? fail(HEDL_ERR_OOM, "device allocation failed")
                                                                : cuda_fail(kb, e, "device allocation");
    kb->allocs.push_back(p);
    kb->device_bytes += bytes;
    if (n) HEDL_CUDA(kb, cudaMemcpyAsync(p, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
    *dst = (T *)p;
    return HEDL_OK;
}

void free_kb(hedl_kb *kb) {
    if (!kb) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(kb->device);
    pool_release_all(kb);
    for (void *p : kb->allocs) dev_free(p);
    cudaSetDevice(prev);
    delete kb;
    live_kb_add(-1);
}

}  // namespace

extern "C" hedl_status hedl_kb_load(const hedl_kb_desc *desc, int device, void *stream, hedl_kb **out) {
    if (!desc || !out) return fail(HEDL_ERR_INVALID_ARG, "null desc/out");
    *out = nullptr;
    // rows padded to 8 words (32 B = one L2 sector) so row segments start on sector boundaries
    const uint32_t N = desc->n_individuals, W = (N + 31) / 32, W4 = (W + 7) & ~7u;
    const uint32_t C = desc->n_concepts, R = desc->n_roles, D = desc->n_data;
    if (R > 32) return fail(HEDL_ERR_INVALID_ARG, "at most 32 roles supported");
    // program nodes store a data property id in 16 bits and operand references a concept id
    // in 29 bits (internal.h CNode.dir, mkref): larger ids would wrap silently
    if (D > 0xffff) return fail(HEDL_ERR_INVALID_ARG, "at most 65535 data properties supported");
    if (C >= (1u << 29)) return fail(HEDL_ERR_INVALID_ARG, "at most 2^29-1 concepts supported");
    if (C && W && !desc->concept_bits) return fail(HEDL_ERR_INVALID_ARG, "concept_bits is null");
    if (R && !desc->role_edge_off) return fail(HEDL_ERR_INVALID_ARG, "role_edge_off is null");
    if (D && !desc->data_off) return fail(HEDL_ERR_INVALID_ARG, "data_off is null");
    const uint32_t S = desc->n_strings;
    if (S > 0xffff) return fail(HEDL_ERR_INVALID_ARG, "at most 65535 string roles supported");
    if (S && !desc->str_off) return fail(HEDL_ERR_INVALID_ARG, "str_off is null");
    if (desc->n_pos && !desc->pos_ids) return fail(HEDL_ERR_INVALID_ARG, "pos_ids is null");
    if (desc->n_neg && !desc->neg_ids) return fail(HEDL_ERR_INVALID_ARG, "neg_ids is null");
    // tail bits of every concept row must be 0
    if (C && W && (N & 31)) {
        const uint32_t tail = ~((1u << (N & 31)) - 1u);
        for (uint32_t c = 0; c < C; ++c)
            if (desc->concept_bits[(uint64_t)c * W + W - 1] & tail)
                return fail(HEDL_ERR_INVALID_ARG, "concept " + std::to_string(c) + " has non-zero tail bits");
    }
    if (R) {
        if (desc->role_edge_off[0] != 0) return fail(HEDL_ERR_INVALID_ARG, "role_edge_off[0] != 0");
        for (uint32_t r = 0; r < R; ++r)
            if (desc->role_edge_off[r + 1] < desc->role_edge_off[r]) return fail(HEDL_ERR_INVALID_ARG, "role_edge_off not monotone");
        if (desc->role_edge_off[R] && (!desc->edge_subj || !desc->edge_obj)) return fail(HEDL_ERR_INVALID_ARG, "edge arrays null");
    }
    if (D) {
        if (desc->data_off[0] != 0) return fail(HEDL_ERR_INVALID_ARG, "data_off[0] != 0");
        for (uint32_t d = 0; d < D; ++d)
            if (desc->data_off[d + 1] < desc->data_off[d]) return fail(HEDL_ERR_INVALID_ARG, "data_off not monotone");
        if (desc->data_off[D] && (!desc->data_subj || !desc->data_val)) return fail(HEDL_ERR_INVALID_ARG, "data arrays null");
    }
    if (S) {
        if (desc->str_off[0] != 0) return fail(HEDL_ERR_INVALID_ARG, "str_off[0] != 0");
        for (uint32_t r = 0; r < S; ++r)
            if (desc->str_off[r + 1] < desc->str_off[r]) return fail(HEDL_ERR_INVALID_ARG, "str_off not monotone");
        const uint64_t A = desc->str_off[S];
        if (A && (!desc->str_subj || !desc->str_val_off)) return fail(HEDL_ERR_INVALID_ARG, "string arrays null");
        if (A) {
            for (uint64_t k = 0; k < A; ++k)
                if (desc->str_val_off[k + 1] < desc->str_val_off[k]) return fail(HEDL_ERR_INVALID_ARG, "str_val_off not monotone");
            if (desc->str_val_off[A] > desc->str_val_off[0] && !desc->str_bytes) return fail(HEDL_ERR_INVALID_ARG, "str_bytes is null");
        }
    }
    // examples (P and N disjoint)
    std::vector<uint32_t> pos(W4, 0), neg(W4, 0);
    for (uint32_t i = 0; i < desc->n_pos; ++i) {
        uint32_t x = desc->pos_ids[i];
        if (x >= N) return fail(HEDL_ERR_OUT_OF_RANGE, "pos id >= N");
        pos[x >> 5] |= 1u << (x & 31);
    }
    for (uint32_t i = 0; i < desc->n_neg; ++i) {
        uint32_t x = desc->neg_ids[i];
        if (x >= N) return fail(HEDL_ERR_OUT_OF_RANGE, "neg id >= N");
        if (pos[x >> 5] & (1u << (x & 31))) return fail(HEDL_ERR_EXAMPLE_CONFLICT, "individual " + std::to_string(x) + " is both + and -");
        neg[x >> 5] |= 1u << (x & 31);
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(HEDL_ERR_UNSUPPORTED, "no such CUDA device");
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return fail(HEDL_ERR_UNSUPPORTED, "device query failed");
    if (prop.major != 10) return fail(HEDL_ERR_UNSUPPORTED, "library is built for sm_100a (B200) only");

    // ---- host build ------------------------------------------------------------
    std::vector<HostCSR> fw(R), tr(R);
    for (uint32_t r = 0; r < R; ++r) {
        const uint64_t a = desc->role_edge_off[r], b = desc->role_edge_off[r + 1];
        hedl_status st = build_forward(N, desc->edge_subj + a, desc->edge_obj + a, b - a, fw[r]);
        if (st) return st;
        build_transpose(N, fw[r], tr[r]);
    }
    struct HostData { std::vector<uint32_t> row_ptr; std::vector<float> val; };
    std::vector<HostData> hd(D);
    for (uint32_t d = 0; d < D; ++d) {
        const uint64_t a = desc->data_off[d], b = desc->data_off[d + 1];
        std::vector<uint64_t> cnt(N + 1, 0);
        for (uint64_t k = a; k < b; ++k) {
            if (desc->data_subj[k] >= N) return fail(HEDL_ERR_OUT_OF_RANGE, "data subject id >= N");
            if (!std::isnan(desc->data_val[k])) cnt[desc->data_subj[k] + 1]++;   // NaN never matches (Q10)
        }
        for (uint32_t i = 0; i < N; ++i) cnt[i + 1] += cnt[i];
        if (cnt[N] > 0xffffffffull) return fail(HEDL_ERR_INVALID_ARG, "data property has >= 2^32 values");
        hd[d].row_ptr.resize(N + 1);
        for (uint32_t i = 0; i <= N; ++i) hd[d].row_ptr[i] = (uint32_t)cnt[i];
        hd[d].val.resize(cnt[N]);
        std::vector<uint64_t> p(cnt.begin(), cnt.end() - 1);
        for (uint64_t k = a; k < b; ++k)
            if (!std::isnan(desc->data_val[k])) hd[d].val[p[desc->data_subj[k]]++] = desc->data_val[k];
        auto &v = hd[d].val;
        auto &rp = hd[d].row_ptr;
        parallel_ranges(N, [&](uint64_t x0, uint64_t x1) {
            for (uint64_t i = x0; i < x1; ++i) std::sort(v.begin() + rp[i], v.begin() + rp[i + 1]);
        });
    }

    // string roles: intern the distinct values of each role (stringValuesMapping),
    // then a CSR subject -> ascending distinct value ids (duplicate pairs removed)
    struct HostStr {
        std::vector<uint32_t> row_ptr, vid;
        std::vector<uint64_t> dict_off;
        std::vector<uint8_t> dict;
        std::unordered_map<std::string, uint32_t> ids;
    };
    std::vector<HostStr> hs(S);
    for (uint32_t r = 0; r < S; ++r) {
        HostStr &H = hs[r];
        const uint64_t a = desc->str_off[r], b = desc->str_off[r + 1];
        std::vector<uint32_t> kv(b - a);
        H.dict_off.push_back(0);
        for (uint64_t k = a; k < b; ++k) {
            if (desc->str_subj[k] >= N) return fail(HEDL_ERR_OUT_OF_RANGE, "string subject id >= N");
            const uint64_t v0 = desc->str_val_off[k], v1 = desc->str_val_off[k + 1];
            std::string key((const char *)desc->str_bytes + v0, (const char *)desc->str_bytes + v1);
            auto it = H.ids.find(key);
            if (it == H.ids.end()) {
                if (H.ids.size() >= 0xffffffffull) return fail(HEDL_ERR_INVALID_ARG, "string role has >= 2^32 values");
                it = H.ids.emplace(std::move(key), (uint32_t)H.ids.size()).first;
                H.dict.insert(H.dict.end(), desc->str_bytes + v0, desc->str_bytes + v1);
                H.dict_off.push_back(H.dict.size());
            }
            kv[k - a] = it->second;
        }
        std::vector<uint32_t> subj(desc->str_subj + a, desc->str_subj + b);
        HostCSR c;
        hedl_status st = build_forward(N, subj.data(), kv.data(), b - a, c, H.ids.size());
        if (st) return st;
        H.row_ptr.swap(c.row_ptr);
        H.vid.swap(c.col);
    }

    // ---- upload -------------------------------------------------------------------
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    if (cudaSetDevice(device) != cudaSuccess) return fail(HEDL_ERR_CUDA, "cudaSetDevice failed");
    cudaStream_t st = (cudaStream_t)stream;
    hedl_kb *kb = new hedl_kb();
    live_kb_add(1);
    kb->device = device;
    kb->sm_count = prop.multiProcessorCount;
    kb->N = N; kb->W = W; kb->W4 = W4; kb->C = C; kb->R = R; kb->D = D;
    auto bail = [&](hedl_status s) { free_kb(kb); cudaSetDevice(prev_dev); return s; };
    hedl_status s;
    {
        std::vector<uint32_t> cpad((uint64_t)C * W4, 0);
        for (uint32_t c = 0; c < C; ++c)
            if (W) std::memcpy(&cpad[(uint64_t)c * W4], desc->concept_bits + (uint64_t)c * W, W * 4ull);
        std::vector<uint32_t> ones(W4, 0), zeros(W4, 0);
        for (uint32_t w = 0; w < W; ++w) ones[w] = 0xffffffffu;
        if (W && (N & 31)) ones[W - 1] = (1u << (N & 31)) - 1u;
        if ((s = upload(kb, st, &kb->concepts, cpad.data(), cpad.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->ones, ones.data(), ones.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->zeros, zeros.data(), zeros.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->pos, pos.data(), pos.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->neg, neg.data(), neg.size()))) return bail(s);
        for (uint32_t w = 0; w < W4; ++w) { kb->npos += __builtin_popcount(pos[w]); kb->nneg += __builtin_popcount(neg[w]); }
        // example projection: E = P u N in id order; rank r <-> r-th example
        std::vector<uint32_t> exm(W4, 0), exb(W4, 0), ex;
        uint32_t rank = 0;
        for (uint32_t w = 0; w < W4; ++w) {
            exm[w] = pos[w] | neg[w];
            exb[w] = rank;
            for (uint32_t m = exm[w]; m; m &= m - 1) ex.push_back(32 * w + __builtin_ctz(m));
            rank += __builtin_popcount(exm[w]);
        }
        kb->M = rank;
        kb->h_ex = ex;
        kb->MW = (rank + 31) / 32;
        kb->MW4 = (kb->MW + 3) & ~3u;
        const uint32_t MW4 = kb->MW4;
        std::vector<uint32_t> pc((uint64_t)C * MW4, 0), pon(MW4, 0), pp(MW4, 0), pn(MW4, 0);
        for (uint32_t r = 0; r < rank; ++r) {
            const uint32_t x = ex[r], bit = 1u << (r & 31);
            pon[r >> 5] |= bit;
            if (pos[x >> 5] >> (x & 31) & 1u) pp[r >> 5] |= bit;
            if (neg[x >> 5] >> (x & 31) & 1u) pn[r >> 5] |= bit;
            for (uint32_t c = 0; c < C; ++c)
                if (desc->concept_bits[(uint64_t)c * W + (x >> 5)] >> (x & 31) & 1u) pc[(uint64_t)c * MW4 + (r >> 5)] |= bit;
        }
        if ((s = upload(kb, st, &kb->ex_mask, exm.data(), exm.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->ex_ids, ex.data(), ex.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->ex_base, exb.data(), exb.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->pconcepts, pc.data(), pc.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->pones, pon.data(), pon.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->ppos, pp.data(), pp.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->pneg, pn.data(), pn.size()))) return bail(s);
        if (cudaStreamSynchronize(st) != cudaSuccess) return bail(fail(HEDL_ERR_CUDA, "upload failed"));
    }
    // U_d per direction (the distinct neighbours of the example rows, in id order): the rows of
    // the U sweeps, built with every direction below
    std::vector<std::vector<uint32_t>> ulists;
    if (kb->M && 2 * R <= kMaxUDirs) {
        ulists.resize(2 * R);
        std::vector<uint8_t> mark(N);
        for (uint32_t d = 0; d < 2 * R; ++d) {
            const HostCSR &h = (d & 1) ? tr[d >> 1] : fw[d >> 1];
            std::fill(mark.begin(), mark.end(), 0);
            for (uint32_t x : kb->h_ex)
                for (uint32_t e = h.row_ptr[x]; e < h.row_ptr[x + 1]; ++e) mark[h.col[e]] = 1;
            for (uint32_t y = 0; y < N; ++y)
                if (mark[y]) ulists[d].push_back(y);
        }
    }
    kb->dirs.resize(2 * R);
    kb->dir_bytes.resize(2 * R);
    for (uint32_t r = 0; r < R; ++r) {
        for (int inv = 0; inv < 2; ++inv) {
            HostCSR &h = inv ? tr[r] : fw[r];
            hedl_dir &dr = kb->dirs[2 * r + inv];
            dr.E = h.col.size();
            if ((s = upload(kb, st, &dr.row_ptr, h.row_ptr.data(), h.row_ptr.size()))) return bail(s);
            if ((s = upload(kb, st, &dr.col, h.col.data(), h.col.size()))) return bail(s);
            std::vector<uint32_t> hx, hn;
            std::vector<uint4> chunks;
            uint64_t eh = 0;                               // heavy edges: sizes the chunks
            for (uint32_t x = 0; x < N; ++x)
                if (h.row_ptr[x + 1] - h.row_ptr[x] > kHeavyDeg) eh += h.row_ptr[x + 1] - h.row_ptr[x];
            const uint32_t hc = heavy_chunk(eh, kb->sm_count);
            for (uint32_t x = 0; x < N; ++x) {
                const uint32_t a = h.row_ptr[x], b = h.row_ptr[x + 1], deg = b - a;
                dr.max_deg = std::max(dr.max_deg, deg);
                if (deg > kHeavyDeg) {
                    const uint32_t hi = (uint32_t)hx.size();
                    hx.push_back(x);
                    uint32_t nc = 0;
                    for (uint32_t e = a; e < b; e += hc, ++nc)
                        chunks.push_back(make_uint4(hi, e, std::min(b, e + hc), 0));
                    hn.push_back(nc);
                    dr.E_heavy += deg;
                }
            }
            // lane-packed path: per tile of 1024 rows, medium rows then light rows, degree-descending
            dr.n_tiles = (N + 1023) / 1024;
            std::vector<uint4> tiles(dr.n_tiles + 1);
            std::vector<uint32_t> order;
            order.reserve(N - hx.size());
            {
                uint32_t hpos = 0;
                std::vector<uint32_t> med, light;
                for (uint32_t t = 0; t < dr.n_tiles; ++t) {
                    med.clear();
                    light.clear();
                    const uint32_t xa = t * 1024, xb = std::min(N, xa + 1024);
                    while (hpos < hx.size() && hx[hpos] < xa) ++hpos;
                    tiles[t].w = hpos;
                    for (uint32_t x = xa; x < xb; ++x) {
                        const uint32_t deg = h.row_ptr[x + 1] - h.row_ptr[x];
                        if (deg > kHeavyDeg) continue;
                        (deg > kLightDeg ? med : light).push_back(x);
                    }
                    auto by_deg = [&](uint32_t a, uint32_t b) {
                        const uint32_t da = h.row_ptr[a + 1] - h.row_ptr[a], db = h.row_ptr[b + 1] - h.row_ptr[b];
                        return da != db ? da > db : a < b;
                    };
                    std::sort(med.begin(), med.end(), by_deg);
                    std::sort(light.begin(), light.end(), by_deg);
                    tiles[t].x = (uint32_t)order.size();
                    tiles[t].y = (uint32_t)med.size();
                    tiles[t].z = (uint32_t)light.size();
                    order.insert(order.end(), med.begin(), med.end());
                    order.insert(order.end(), light.begin(), light.end());
                }
                tiles[dr.n_tiles] = make_uint4((uint32_t)order.size(), 0, 0, (uint32_t)hx.size());
            }
            if ((s = upload(kb, st, &dr.tiles, tiles.data(), tiles.size()))) return bail(s);
            if ((s = upload(kb, st, &dr.order, order.data(), order.size()))) return bail(s);
            {
                // tiles in decreasing sweep cost (edges of their light and medium rows + a fixed
                // share for the transpose-back): the persistent tile kernel takes them in this
                // order, so the longest tiles start first (LPT) and the tail is short
                std::vector<uint64_t> cost(dr.n_tiles);
                std::vector<uint32_t> rank(dr.n_tiles);
                for (uint32_t t = 0; t < dr.n_tiles; ++t) {
                    uint64_t c = 2048;
                    for (uint32_t i = tiles[t].x; i < tiles[t + 1].x; ++i)
                        c += h.row_ptr[order[i] + 1] - h.row_ptr[order[i]];
                    cost[t] = c;
                    rank[t] = t;
                }
                std::stable_sort(rank.begin(), rank.end(), [&](uint32_t a, uint32_t b) { return cost[a] > cost[b]; });
                if (dr.n_tiles && (s = upload(kb, st, &dr.tile_rank, rank.data(), rank.size()))) return bail(s);
                // medium rows are degree-descending: the big ones (deg > kMidDeg) come first
                std::vector<uint32_t> nbig(dr.n_tiles);
                for (uint32_t t = 0; t < dr.n_tiles; ++t) {
                    uint32_t nb = 0;
                    for (uint32_t i = tiles[t].x; i < tiles[t].x + tiles[t].y; ++i)
                        nb += h.row_ptr[order[i] + 1] - h.row_ptr[order[i]] > kMidDeg;
                    nbig[t] = nb;
                }
                if (dr.n_tiles && (s = upload(kb, st, &dr.tile_nbig, nbig.data(), nbig.size()))) return bail(s);
            }
            {
                std::vector<uint32_t> tslice(dr.n_tiles + 1), soff, sw, scol;
                for (uint32_t t = 0; t < dr.n_tiles; ++t) {
                    tslice[t] = (uint32_t)soff.size();
                    const uint32_t l0 = tiles[t].x + tiles[t].y, nl = tiles[t].z;
                    for (uint32_t a = 0; a < nl; a += 16) {
                        const uint32_t x0 = order[l0 + a];
                        // rows sorted: the first is widest; width padded to a multiple of 4 (4 gathers per step)
                        const uint32_t wdt = (h.row_ptr[x0 + 1] - h.row_ptr[x0] + 3) & ~3u;
                        soff.push_back((uint32_t)scol.size());
                        sw.push_back(wdt);
                        const size_t b = scol.size();
                        scol.resize(b + (size_t)wdt * 16, 0xffffffffu);
                        for (uint32_t i = 0; i < 16 && a + i < nl; ++i) {
                            const uint32_t x = order[l0 + a + i];
                            for (uint32_t k = 0, e = h.row_ptr[x]; e < h.row_ptr[x + 1]; ++e, ++k)
                                scol[b + (size_t)k * 16 + i] = h.col[e];
                        }
                    }
                }
                tslice[dr.n_tiles] = (uint32_t)soff.size();
                if (scol.size() >= 0xffffffffull) return bail(fail(HEDL_ERR_UNSUPPORTED, "SELL layout too large"));
                if ((s = upload(kb, st, &dr.tile_slice, tslice.data(), tslice.size()))) return bail(s);
                soff.push_back((uint32_t)scol.size());    // sentinel: slice s spans [sell_off[s], sell_off[s + 1])
                if ((s = upload(kb, st, &dr.sell_off, soff.data(), soff.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.sell_w, sw.data(), sw.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.sell_col, scol.data(), scol.size()))) return bail(s);
                if (cudaStreamSynchronize(st) != cudaSuccess) return bail(fail(HEDL_ERR_CUDA, "upload failed"));
            }
            // EX packs: example rows only (ranks of E), blocks of 128 ranks
            {
                const std::vector<uint32_t> &ex = kb->h_ex;
                const uint32_t M = (uint32_t)ex.size();
                // example-row CSR over ranks with neighbours as compact T indices (U = distinct
                // neighbours of the example rows, in id order)
                std::vector<uint32_t> erp(M + 1, 0);
                for (uint32_t r = 0; r < M; ++r) erp[r + 1] = erp[r] + (h.row_ptr[ex[r] + 1] - h.row_ptr[ex[r]]);
                std::vector<uint32_t> umask(W4, 0), ubase(W4, 0), ecol(erp[M]);
                for (uint32_t r = 0; r < M; ++r)
                    for (uint32_t e = h.row_ptr[ex[r]]; e < h.row_ptr[ex[r] + 1]; ++e) {
                        const uint32_t y = h.col[e];
                        umask[y >> 5] |= 1u << (y & 31);
                    }
                uint32_t nu = 0;
                for (uint32_t w = 0; w < W4; ++w) {
                    ubase[w] = nu;
                    nu += (uint32_t)__builtin_popcount(umask[w]);
                }
                for (uint32_t r = 0; r < M; ++r)
                    for (uint32_t e = h.row_ptr[ex[r]], k = erp[r]; e < h.row_ptr[ex[r] + 1]; ++e, ++k) {
                        const uint32_t y = h.col[e];
                        ecol[k] = ubase[y >> 5] + (uint32_t)__builtin_popcount(umask[y >> 5] & ((1u << (y & 31)) - 1u));
                    }
                dr.n_u = nu;
                dr.UW = (nu + 31) / 32;
                dr.UW4 = (dr.UW + 7) & ~7u;
                {
                    std::vector<uint32_t> ul;
                    ul.reserve(nu);
                    for (uint32_t w = 0; w < W4; ++w)
                        for (uint32_t m = umask[w]; m; m &= m - 1) ul.push_back(32 * w + __builtin_ctz(m));
                    std::vector<uint32_t> uc((uint64_t)C * dr.UW4, 0), uon(dr.UW4, 0);
                    for (uint32_t t = 0; t < nu; ++t) {
                        const uint32_t y = ul[t], bit = 1u << (t & 31);
                        uon[t >> 5] |= bit;
                        for (uint32_t c = 0; c < C; ++c)
                            if (desc->concept_bits[(uint64_t)c * W + (y >> 5)] >> (y & 31) & 1u) uc[(uint64_t)c * dr.UW4 + (t >> 5)] |= bit;
                    }
                    if ((s = upload(kb, st, &dr.uconcepts, uc.data(), uc.size()))) return bail(s);
                    if ((s = upload(kb, st, &dr.uones, uon.data(), uon.size()))) return bail(s);
                    if ((s = upload(kb, st, &dr.ulist, ul.data(), ul.size()))) return bail(s);
                    if (cudaStreamSynchronize(st) != cudaSuccess) return bail(fail(HEDL_ERR_CUDA, "upload failed"));
                }
                if ((s = upload(kb, st, &dr.ex_rp, erp.data(), erp.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.ex_ccol, ecol.data(), ecol.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.ex_umask, umask.data(), umask.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.ex_ubase, ubase.data(), ubase.size()))) return bail(s);
                dr.n_ex_blocks = (M + 127) / 128;
                std::vector<uint4> et(dr.n_ex_blocks + 1);
                std::vector<uint32_t> eo, ehx, ehr, ehn;
                std::vector<uint4> ech;
                std::vector<uint32_t> med, light;
                auto degr = [&](uint32_t r) { return h.row_ptr[ex[r] + 1] - h.row_ptr[ex[r]]; };
                uint64_t ehe = 0;
                for (uint32_t r = 0; r < M; ++r)
                    if (degr(r) > kHeavyDeg) ehe += degr(r);
                const uint32_t ehc = heavy_chunk(ehe, kb->sm_count);
                for (uint32_t b = 0; b < dr.n_ex_blocks; ++b) {
                    med.clear();
                    light.clear();
                    et[b].w = (uint32_t)ehx.size();
                    for (uint32_t r = b * 128; r < std::min(M, b * 128 + 128); ++r) {
                        const uint32_t d = degr(r);
                        if (d > kHeavyDeg) {
                            const uint32_t hi = (uint32_t)ehx.size();
                            ehx.push_back(ex[r]);
                            ehr.push_back(r);
                            const uint32_t a = erp[r], e = erp[r + 1];     // in the example-row CSR
                            uint32_t nc = 0;
                            for (uint32_t q = a; q < e; q += ehc, ++nc)
                                ech.push_back(make_uint4(hi, q, std::min(e, q + ehc), 0));
                            ehn.push_back(nc);
                            dr.E_ex_heavy += d;
                        } else {
                            (d > kLightDeg ? med : light).push_back(r);
                            dr.E_ex += d;
                        }
                    }
                    auto by_deg = [&](uint32_t a, uint32_t c) { return degr(a) != degr(c) ? degr(a) > degr(c) : a < c; };
                    std::sort(med.begin(), med.end(), by_deg);
                    std::sort(light.begin(), light.end(), by_deg);
                    et[b].x = (uint32_t)eo.size();
                    et[b].y = (uint32_t)med.size();
                    et[b].z = (uint32_t)light.size();
                    eo.insert(eo.end(), med.begin(), med.end());
                    eo.insert(eo.end(), light.begin(), light.end());
                }
                et[dr.n_ex_blocks] = make_uint4((uint32_t)eo.size(), 0, 0, (uint32_t)ehx.size());
                dr.n_ex_heavy = (uint32_t)ehx.size();
                dr.n_ex_chunks = (uint32_t)ech.size();
                if ((s = upload(kb, st, &dr.ex_tiles, et.data(), et.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.ex_order, eo.data(), eo.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.ex_hx, ehx.data(), ehx.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.ex_hrank, ehr.data(), ehr.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.ex_hn, ehn.data(), ehn.size()))) return bail(s);
                if ((s = upload(kb, st, &dr.ex_chunks, ech.data(), ech.size()))) return bail(s);
                if (cudaStreamSynchronize(st) != cudaSuccess) return bail(fail(HEDL_ERR_CUDA, "upload failed"));
            }
            // U sweeps of this direction: its rows restricted to U_d' for every d'
            for (uint32_t du = 0; du < ulists.size(); ++du) {
                const std::vector<uint32_t> &rows = ulists[du];
                hedl_rowset &rs = dr.usw[du];
                const uint32_t n = (uint32_t)rows.size();
                rs.n_rows = n;
                rs.n_blocks = (n + 127) / 128;
                std::vector<uint32_t> rp(n + 1, 0), cl;
                for (uint32_t q = 0; q < n; ++q) rp[q + 1] = rp[q] + (h.row_ptr[rows[q] + 1] - h.row_ptr[rows[q]]);
                cl.reserve(rp[n]);
                for (uint32_t q = 0; q < n; ++q)
                    for (uint32_t e = h.row_ptr[rows[q]]; e < h.row_ptr[rows[q] + 1]; ++e) cl.push_back(h.col[e]);
                std::vector<uint4> tb(rs.n_blocks + 1), chs;
                std::vector<uint32_t> ord, rhx, rhr, rhn, med, light;
                auto deg = [&](uint32_t q) { return rp[q + 1] - rp[q]; };
                uint64_t rhe = 0;
                for (uint32_t q = 0; q < n; ++q)
                    if (deg(q) > kHeavyDeg) rhe += deg(q);
                const uint32_t rhc = heavy_chunk(rhe, kb->sm_count);
                for (uint32_t b = 0; b < rs.n_blocks; ++b) {
                    med.clear();
                    light.clear();
                    tb[b].w = (uint32_t)rhx.size();
                    for (uint32_t q = b * 128; q < std::min(n, b * 128 + 128); ++q) {
                        const uint32_t dq = deg(q);
                        if (dq > kHeavyDeg) {
                            const uint32_t hi = (uint32_t)rhx.size();
                            rhx.push_back(rows[q]);
                            rhr.push_back(q);
                            uint32_t nc = 0;
                            for (uint32_t e = rp[q]; e < rp[q + 1]; e += rhc, ++nc)
                                chs.push_back(make_uint4(hi, e, std::min(rp[q + 1], e + rhc), 0));
                            rhn.push_back(nc);
                            rs.E_heavy += dq;
                        } else {
                            (dq > kLightDeg ? med : light).push_back(q);
                            rs.E += dq;
                        }
                    }
                    auto by_deg = [&](uint32_t a, uint32_t c) { return deg(a) != deg(c) ? deg(a) > deg(c) : a < c; };
                    std::sort(med.begin(), med.end(), by_deg);
                    std::sort(light.begin(), light.end(), by_deg);
                    tb[b].x = (uint32_t)ord.size();
                    tb[b].y = (uint32_t)med.size();
                    tb[b].z = (uint32_t)light.size();
                    ord.insert(ord.end(), med.begin(), med.end());
                    ord.insert(ord.end(), light.begin(), light.end());
                }
                tb[rs.n_blocks] = make_uint4((uint32_t)ord.size(), 0, 0, (uint32_t)rhx.size());
                rs.n_heavy = (uint32_t)rhx.size();
                rs.n_chunks = (uint32_t)chs.size();
                rs.frac = h.col.empty() ? 1.0 : (double)(rs.E + rs.E_heavy) / (double)h.col.size();
                if ((s = upload(kb, st, &rs.rp, rp.data(), rp.size()))) return bail(s);
                if ((s = upload(kb, st, &rs.col, cl.data(), cl.size()))) return bail(s);
                if ((s = upload(kb, st, &rs.tiles, tb.data(), tb.size()))) return bail(s);
                if ((s = upload(kb, st, &rs.order, ord.data(), ord.size()))) return bail(s);
                if ((s = upload(kb, st, &rs.hx, rhx.data(), rhx.size()))) return bail(s);
                if ((s = upload(kb, st, &rs.hrank, rhr.data(), rhr.size()))) return bail(s);
                if ((s = upload(kb, st, &rs.hn, rhn.data(), rhn.size()))) return bail(s);
                if ((s = upload(kb, st, &rs.chunks, chs.data(), chs.size()))) return bail(s);
                if (cudaStreamSynchronize(st) != cudaSuccess) return bail(fail(HEDL_ERR_CUDA, "upload failed"));
            }
            dr.n_heavy = (uint32_t)hx.size();
            dr.n_chunks = (uint32_t)chunks.size();
            if ((s = upload(kb, st, &dr.heavy_x, hx.data(), hx.size()))) return bail(s);
            if ((s = upload(kb, st, &dr.heavy_nchunks, hn.data(), hn.size()))) return bail(s);
            if ((s = upload(kb, st, &dr.chunks, chunks.data(), chunks.size()))) return bail(s);
            kb->dir_bytes[2 * r + inv] = 4.0 * (N + 1) + 4.0 * dr.E;
            // the uploads read host vectors that die at scope end: wait before reuse
            if (cudaStreamSynchronize(st) != cudaSuccess) return bail(fail(HEDL_ERR_CUDA, "upload failed"));
            dr.h_row_ptr = std::move(h.row_ptr);
            std::vector<uint32_t>().swap(h.col);
        }
    }
    kb->data.resize(D);
    kb->data_bytes.resize(D);
    for (uint32_t d = 0; d < D; ++d) {
        kb->data[d].V = hd[d].val.size();
        if ((s = upload(kb, st, &kb->data[d].row_ptr, hd[d].row_ptr.data(), hd[d].row_ptr.size()))) return bail(s);
        if ((s = upload(kb, st, &kb->data[d].val, hd[d].val.data(), hd[d].val.size()))) return bail(s);
        kb->data_bytes[d] = 4.0 * (N + 1) + 4.0 * kb->data[d].V;
        if (cudaStreamSynchronize(st) != cudaSuccess) return bail(fail(HEDL_ERR_CUDA, "upload failed"));
    }
    kb->S = S;
    kb->sdirs.resize(S);
    kb->str_bytes.resize(S);
    for (uint32_t r = 0; r < S; ++r) {
        hedl_sdir &sd = kb->sdirs[r];
        HostStr &H = hs[r];
        sd.E = H.vid.size();
        sd.V = H.ids.size();
        sd.dict_bytes = H.dict.size();
        if ((s = upload(kb, st, &sd.row_ptr, H.row_ptr.data(), H.row_ptr.size()))) return bail(s);
        if ((s = upload(kb, st, &sd.vid, H.vid.data(), H.vid.size()))) return bail(s);
        if ((s = upload(kb, st, &sd.dict_off, H.dict_off.data(), H.dict_off.size()))) return bail(s);
        if ((s = upload(kb, st, &sd.dict, H.dict.data(), H.dict.size()))) return bail(s);
        kb->str_bytes[r] = 4.0 * (N + 1) + 4.0 * sd.E;
        if (cudaStreamSynchronize(st) != cudaSuccess) return bail(fail(HEDL_ERR_CUDA, "upload failed"));
        sd.ids.swap(H.ids);
    }
    cudaSetDevice(prev_dev);
    *out = kb;
    return HEDL_OK;
}

namespace hedl {
void kb_release(const hedl_kb *kb) {
    if (kb && const_cast<hedl_kb *>(kb)->refs.fetch_sub(1) == 1) free_kb(const_cast<hedl_kb *>(kb));
}
}  // namespace hedl

// Programs keep their KB alive: the device memory goes when the handle and every
// program compiled against it are freed (in any order).
extern "C" hedl_status hedl_kb_free(hedl_kb *kb) {
    kb_release(kb);
    return HEDL_OK;
}

extern "C" hedl_status hedl_kb_get_info(const hedl_kb *kb, hedl_kb_info *out) {
    if (!kb || !out) return fail(HEDL_ERR_INVALID_ARG, "null kb/out");
    std::memset(out, 0, sizeof(*out));
    out->n_individuals = kb->N; out->words = kb->W; out->words_padded = kb->W4;
    out->n_concepts = kb->C; out->n_roles = kb->R; out->n_data = kb->D;
    out->n_pos = kb->npos; out->n_neg = kb->nneg;
    out->device_bytes = kb->device_bytes;
    for (size_t i = 0; i < kb->dirs.size() && i < 64; ++i) {
        out->edges[i] = kb->dirs[i].E;
        out->heavy[i] = kb->dirs[i].n_heavy;
    }
    out->n_strings = kb->S;
    for (size_t i = 0; i < kb->sdirs.size() && i < 32; ++i) {
        out->str_pairs[i] = kb->sdirs[i].E;
        out->str_values[i] = kb->sdirs[i].V;
    }
    return HEDL_OK;
}

// Per-node sm_100a kernels of the hot path.
//
//  k_bool           n-ary AND/OR with per-operand complement (Alg. 2),
//                   128-bit words, tail mask, fused coverage (Alg. 15).
//  k_restrict_tile  exists / forall / >=n / <=n / =n over a role direction's CSR
//                   (Algs. 4, 6, 8; inverse = transposed CSR):
//                   1,024-row tiles in degree order, light rows from SELL-16 slices,
//                   warp-cooperative medium rows, saturating counts with early exit,
//                   bits assembled in shared memory, fused coverage.
//  k_restrict_heavy heavy rows (deg > kHeavyDeg) split over CTAs; the last CTA
//                   of a row finalises its bit with atomicOr (no other atomics on rows).
//  k_drange         exists d.[lo,hi] over sorted per-individual values (Alg. 10, Q9).
//  k_string         string EQUAL / CONTAIN restrictions (Algs. 11-14).
//
// Every output word is written exactly once by one warp (plus commutative
// atomicOr of heavy bits), so results are deterministic (no paper-style
// check-then-write race).
#include <algorithm>

#include "internal.h"

namespace hedl {

namespace {
constexpr uint32_t FULL = 0xffffffffu;

__device__ __forceinline__ uint32_t probe(const uint32_t *__restrict__ child, uint32_t y, uint32_t cmask) {
    return ((__ldg(child + (y >> 5)) ^ cmask) >> (y & 31)) & 1u;
}

__device__ __forceinline__ bool pred_eval(uint32_t pred, uint32_t cnt, uint32_t n) {
    switch (pred) {
    case P_GE: return cnt >= n;
    case P_LE: return cnt <= n;
    case P_EQ: return cnt == n;
    default: return cnt > 0 && cnt <= n;   // P_LEP: paper MAX
    }
}

__device__ __forceinline__ uint32_t tail_word(uint32_t v, uint32_t w, uint32_t W, uint32_t N) {
    if (w >= W) return 0u;
    if (w == W - 1 && (N & 31u)) v &= (1u << (N & 31u)) - 1u;
    return v;
}

// block-wide reduction of (tp, fp) and one u64 atomic per CTA.  All threads call.
__device__ __forceinline__ void block_cover(hedl_counts *counts, int slot, uint32_t tp, uint32_t fp) {
    __shared__ uint32_t s_tp[32], s_fp[32];
    tp = __reduce_add_sync(FULL, tp);
    fp = __reduce_add_sync(FULL, fp);
    const uint32_t wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { s_tp[wid] = tp; s_fp[wid] = fp; }
    __syncthreads();
    if (wid == 0) {
        const uint32_t nw = blockDim.x >> 5;
        uint32_t a = lane < nw ? s_tp[lane] : 0u, b = lane < nw ? s_fp[lane] : 0u;
        a = __reduce_add_sync(FULL, a);
        b = __reduce_add_sync(FULL, b);
        if (lane == 0) {
            hedl_counts *c = counts + slot;
            if (a) {
                atomicAdd((unsigned long long *)&c->tp, (unsigned long long)a);
                atomicAdd((unsigned long long *)&c->fn, (unsigned long long)(0ull - a));
            }
            if (b) {
                atomicAdd((unsigned long long *)&c->fp, (unsigned long long)b);
                atomicAdd((unsigned long long *)&c->tn, (unsigned long long)(0ull - b));
            }
        }
    }
}

// ------------------------------------------------------------------------------
__global__ void k_cover_init(hedl_counts *c, uint32_t n, uint64_t npos, uint64_t nneg) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) c[i] = hedl_counts{0, 0, npos, nneg};
}

// ------------------------------------------------------------------------------
// Full rows: blockIdx.y = node, blockIdx.x = a slice of its words.  Each thread owns BU
// uint4 words (interleaved by the grid width, so every load instruction is coalesced) and
// issues all BU loads of an operand before combining them; the node's operand table is
// staged in shared memory once, so the operand loop has no dependent global load.
constexpr int kBoolU = 8;
constexpr uint32_t kBoolSmemOps = 64;
// FULL_ROWS: rows over all N individuals (else projected / U rows): the same code, instantiated
// twice so profiles (ncu kernel names) tell the HBM-sized launches from the L2-sized ones
template <bool FULL_ROWS>
__global__ void __launch_bounds__(256) k_bool(KbDev kb, const BoolDesc *__restrict__ descs,
                                              const Operand *__restrict__ ops, hedl_counts *counts) {
    const BoolDesc d = descs[blockIdx.y];
    __shared__ Operand s_ops[kBoolSmemOps];
    for (uint32_t j = threadIdx.x; j < d.op_count && j < kBoolSmemOps; j += blockDim.x) s_ops[j] = ops[d.op_first + j];
    __syncthreads();
    const uint32_t n4 = kb.W4 >> 2;
    const uint32_t gs = gridDim.x * blockDim.x;           // stride between a thread's words
    uint32_t tp = 0, fp = 0;
    // one form for both: OR accumulates v ^ m; AND accumulates the complement, ~v ^ ~m ...
    // = v ^ ~m, and complements at the end (De Morgan), so every operand word costs one LOP3
    const uint32_t flip = d.is_or ? 0u : FULL;
    for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += gs * kBoolU) {
        uint4 acc[kBoolU];
#pragma unroll
        for (int u = 0; u < kBoolU; ++u) acc[u] = make_uint4(0, 0, 0, 0);
        const bool full = i0 + (kBoolU - 1) * gs < n4;
        for (uint32_t j = 0; j < d.op_count; ++j) {
            const Operand o = j < kBoolSmemOps ? s_ops[j] : ops[d.op_first + j];
            const uint4 *src = reinterpret_cast<const uint4 *>(o.ptr);
            const uint32_t m = o.mask ^ flip;
            uint4 v[kBoolU];
            if (full) {
#pragma unroll
                for (int u = 0; u < kBoolU; ++u) v[u] = __ldg(src + i0 + u * gs);
            } else {
#pragma unroll
                for (int u = 0; u < kBoolU; ++u) v[u] = i0 + u * gs < n4 ? __ldg(src + i0 + u * gs) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kBoolU; ++u) {
                acc[u].x |= v[u].x ^ m; acc[u].y |= v[u].y ^ m; acc[u].z |= v[u].z ^ m; acc[u].w |= v[u].w ^ m;
            }
        }
#pragma unroll
        for (int u = 0; u < kBoolU; ++u) {
            const uint32_t i = i0 + u * gs;
            if (i >= n4) break;
            uint4 a = make_uint4(acc[u].x ^ flip, acc[u].y ^ flip, acc[u].z ^ flip, acc[u].w ^ flip);
            const uint32_t w0 = i << 2;
            if (w0 + 4 >= kb.W) {                          // the uint4 holding word W-1 and later
                a.x = tail_word(a.x, w0, kb.W, kb.N);
                a.y = tail_word(a.y, w0 + 1, kb.W, kb.N);
                a.z = tail_word(a.z, w0 + 2, kb.W, kb.N);
                a.w = tail_word(a.w, w0 + 3, kb.W, kb.N);
            }
            if (d.out) reinterpret_cast<uint4 *>(d.out)[i] = a;   // null: root needed for counts only
            if (d.proj) {
                proj_scatter(kb, d.proj, w0, a.x);
                proj_scatter(kb, d.proj, w0 + 1, a.y);
                proj_scatter(kb, d.proj, w0 + 2, a.z);
                proj_scatter(kb, d.proj, w0 + 3, a.w);
            }
            if (d.cover >= 0) {
                const uint4 p = __ldg(reinterpret_cast<const uint4 *>(kb.pos) + i);
                const uint4 q = __ldg(reinterpret_cast<const uint4 *>(kb.neg) + i);
                tp += __popc(a.x & p.x) + __popc(a.y & p.y) + __popc(a.z & p.z) + __popc(a.w & p.w);
                fp += __popc(a.x & q.x) + __popc(a.y & q.y) + __popc(a.z & q.z) + __popc(a.w & q.w);
            }
        }
    }
    if (d.cover >= 0) block_cover(counts, d.cover, tp, fp);
}

// Short rows (example-projected rows, small KBs): one warp per node, nodes strided over a
// persistent grid.  One CTA per node would leave most of a 256-thread CTA idle and make
// the launch CTA-scheduling bound (10^6 root conjunctions of 2.5 KB rows at C4); a warp
// streams the node's k operand rows with 16 B loads, and writes its counts slot whole
// (the node is never split across warps, so no atomics).
constexpr uint32_t kBoolWarpMaxN4 = 1024;     // rows up to 4,096 words

#ifndef HEDL_BOOLW_MINB
#define HEDL_BOOLW_MINB 4
#endif
template <bool FULL_ROWS>
__global__ void __launch_bounds__(256, HEDL_BOOLW_MINB) k_bool_warp(KbDev kb, const BoolDesc *__restrict__ descs, uint32_t n_desc,
                                                   const Operand *__restrict__ ops, hedl_counts *counts,
                                                   uint64_t npos, uint64_t nneg) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t n4 = kb.W4 >> 2;
    const uint32_t stride = gridDim.x * 8;
    uint32_t k = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (k >= n_desc) return;
    // a node's descriptor and its first four operand descriptors are fetched while the warp
    // works on the previous node (the dependent descriptor loads leave the critical path)
    BoolDesc d = descs[k];
    Operand o4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o4[j] = (uint32_t)j < d.op_count ? ops[d.op_first + j] : Operand{nullptr, 0u, 0u};
    for (; k < n_desc; k += stride) {
        const uint32_t kn = k + stride;
        BoolDesc dn{};
        if (kn < n_desc) dn = descs[kn];
        uint32_t tp = 0, fp = 0;
        // the same one-LOP3 form as k_bool (AND = complemented OR of complements); two uint4
        // per lane in flight per operand
        const uint32_t flip = d.is_or ? 0u : FULL;
        for (uint32_t i0 = lane; i0 < n4; i0 += 64) {
            uint4 acc[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
            const bool two = i0 + 32 < n4;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if ((uint32_t)j >= d.op_count) break;
                const uint4 *src = reinterpret_cast<const uint4 *>(o4[j].ptr);
                const uint4 v0 = __ldg(src + i0);
                const uint4 v1 = two ? __ldg(src + i0 + 32) : make_uint4(0, 0, 0, 0);
                const uint32_t m = o4[j].mask ^ flip;
                acc[0].x |= v0.x ^ m; acc[0].y |= v0.y ^ m; acc[0].z |= v0.z ^ m; acc[0].w |= v0.w ^ m;
                acc[1].x |= v1.x ^ m; acc[1].y |= v1.y ^ m; acc[1].z |= v1.z ^ m; acc[1].w |= v1.w ^ m;
            }
            for (uint32_t j = 4; j < d.op_count; ++j) {
                const Operand o = ops[d.op_first + j];
                const uint4 *src = reinterpret_cast<const uint4 *>(o.ptr);
                const uint4 v0 = __ldg(src + i0);
                const uint4 v1 = two ? __ldg(src + i0 + 32) : make_uint4(0, 0, 0, 0);
                const uint32_t m = o.mask ^ flip;
                acc[0].x |= v0.x ^ m; acc[0].y |= v0.y ^ m; acc[0].z |= v0.z ^ m; acc[0].w |= v0.w ^ m;
                acc[1].x |= v1.x ^ m; acc[1].y |= v1.y ^ m; acc[1].z |= v1.z ^ m; acc[1].w |= v1.w ^ m;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t i = i0 + 32 * h;
                if (h && !two) break;
                uint4 a = acc[h];
                a.x ^= flip; a.y ^= flip; a.z ^= flip; a.w ^= flip;
                const uint32_t w0 = i << 2;
                if (w0 + 4 >= kb.W) {                      // the uint4 holding word W-1 and later
                    a.x = tail_word(a.x, w0, kb.W, kb.N);
                    a.y = tail_word(a.y, w0 + 1, kb.W, kb.N);
                    a.z = tail_word(a.z, w0 + 2, kb.W, kb.N);
                    a.w = tail_word(a.w, w0 + 3, kb.W, kb.N);
                }
                if (d.out) reinterpret_cast<uint4 *>(d.out)[i] = a;
                if (d.proj) {
                    proj_scatter(kb, d.proj, w0, a.x);
                    proj_scatter(kb, d.proj, w0 + 1, a.y);
                    proj_scatter(kb, d.proj, w0 + 2, a.z);
                    proj_scatter(kb, d.proj, w0 + 3, a.w);
                }
                if (d.cover >= 0) {
                    const uint4 p = __ldg(reinterpret_cast<const uint4 *>(kb.pos) + i);
                    const uint4 q = __ldg(reinterpret_cast<const uint4 *>(kb.neg) + i);
                    tp += __popc(a.x & p.x) + __popc(a.y & p.y) + __popc(a.z & p.z) + __popc(a.w & p.w);
                    fp += __popc(a.x & q.x) + __popc(a.y & q.y) + __popc(a.z & q.z) + __popc(a.w & q.w);
                }
            }
        }
        if (d.cover >= 0) {
            tp = __reduce_add_sync(FULL, tp);
            fp = __reduce_add_sync(FULL, fp);
            if (lane == 0) counts[d.cover] = hedl_counts{tp, fp, npos - tp, nneg - fp};
        }
        if (kn < n_desc) {
#pragma unroll
            for (int j = 0; j < 4; ++j) o4[j] = (uint32_t)j < dn.op_count ? ops[dn.op_first + j] : Operand{nullptr, 0u, 0u};
            d = dn;
        }
    }
}

// ------------------------------------------------------------------------------
// per-node restriction over 1,024-row tiles (blockIdx.x = tile, blockIdx.y = node):
// rows in the tile's degree-descending order (no divergence between a warp's rows),
// medium rows warp-cooperative, light rows from the SELL-16 slices (coalesced
// neighbour indices, a lane pair per row taking alternate neighbours), results as
// bits in shared memory, one store per output word.  Heavy rows: k_restrict_heavy.
__global__ void __launch_bounds__(256) k_restrict_tile(KbDev kb, DirDev dir, const RestrictDesc *__restrict__ descs,
                                                       hedl_counts *counts, const uint32_t *__restrict__ push_mode,
                                                       uint32_t push_stride) {
    if (push_mode && push_mode[(size_t)blockIdx.y * push_stride]) return;   // evaluated by the push kernels
    const RestrictDesc d = descs[blockIdx.y];
    __shared__ uint32_t sbits[32];
    const uint32_t t = blockIdx.x, x0 = t * 1024;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x < 32) sbits[threadIdx.x] = 0;
    __syncthreads();
    const uint4 ti = dir.tiles[t];
    const uint32_t sat = d.sat;
    for (uint32_t m = wid; m < ti.y; m += 8) {            // medium rows: warp per row
        const uint32_t x = __ldg(dir.order + ti.x + m);
        const uint32_t a = __ldg(dir.row_ptr + x), b = __ldg(dir.row_ptr + x + 1);
        uint32_t c = 0;
        for (uint32_t e = a; e < b && c < sat; e += 128) {
            uint32_t bit[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t k = e + u * 32 + lane;
                bit[u] = k < b ? probe(d.child, __ldg(dir.col + k), d.cmask) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) c += __popc(__ballot_sync(FULL, bit[u]));
        }
        if (lane == 0 && pred_eval(d.pred, min(c, sat), d.n))
            atomicOr(&sbits[(x - x0) >> 5], 1u << ((x - x0) & 31));
    }
    // light rows: SELL-16 slices
    const uint32_t sbeg = __ldg(dir.tile_slice + t), send = __ldg(dir.tile_slice + t + 1);
    // a thread per row (as the narrow lane packs): the warp's halves take two slices, every
    // thread a row of each of two slice pairs, so four slices' dependent load chains (row
    // order, slice bounds, neighbour ids, probes) overlap per warp step; no pair reduction,
    // and a row stops at its own saturation
    for (uint32_t sl = sbeg + 2 * wid + (lane >> 4); sl < send; sl += 32) {
        uint32_t x[2], w[2], c[2];
        const uint32_t *cp[2];
        bool rv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t s2 = sl + 16 * h;
            const bool sv = s2 < send;
            const uint32_t li = (s2 - sbeg) * 16 + (lane & 15);
            rv[h] = sv && li < ti.z;
            x[h] = rv[h] ? __ldg(dir.order + ti.x + ti.y + li) : 0u;
            cp[h] = sv ? dir.sell_col + __ldg(dir.sell_off + s2) + (lane & 15) : nullptr;
            w[h] = sv ? __ldg(dir.sell_w + s2) : 0u;
            c[h] = 0;
        }
        const uint32_t wm = max(w[0], w[1]);
        for (uint32_t k = 0; k < wm && (c[0] < sat || c[1] < sat); k += 4) {
            uint32_t y[2][4];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    y[h][u] = k + u < w[h] && c[h] < sat ? __ldg(cp[h] + (k + u) * 16) : 0xffffffffu;
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (y[h][u] != 0xffffffffu) c[h] += probe(d.child, y[h][u], d.cmask);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
            if (rv[h] && pred_eval(d.pred, min(c[h], sat), d.n))
                atomicOr(&sbits[(x[h] - x0) >> 5], 1u << ((x[h] - x0) & 31));
    }
    __syncthreads();
    if (wid == 0) {
        const uint32_t w = t * 32 + lane;
        uint32_t tp = 0, fp = 0;
        if (w < kb.W4) {
            const uint32_t word = sbits[lane];            // rows >= N were never set
            if (d.out) d.out[w] = word;
            if (d.proj && w < kb.W) proj_scatter(kb, d.proj, w, word);
            if (d.cover >= 0) {
                tp = __popc(word & __ldg(kb.pos + w));
                fp = __popc(word & __ldg(kb.neg + w));
            }
        }
        if (d.cover >= 0) {
            tp = __reduce_add_sync(FULL, tp);
            fp = __reduce_add_sync(FULL, fp);
            if (lane == 0) {
                hedl_counts *cc = counts + d.cover;
                if (tp) {
                    atomicAdd((unsigned long long *)&cc->tp, (unsigned long long)tp);
                    atomicAdd((unsigned long long *)&cc->fn, 0ull - tp);
                }
                if (fp) {
                    atomicAdd((unsigned long long *)&cc->fp, (unsigned long long)fp);
                    atomicAdd((unsigned long long *)&cc->tn, 0ull - fp);
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------
// heavy rows: blockIdx.x = chunk of <= kHeavyChunk edges, blockIdx.y = node.
__global__ void __launch_bounds__(256) k_restrict_heavy(KbDev kb, DirDev dir, const RestrictDesc *__restrict__ descs,
                                                        hedl_counts *counts, uint32_t *scratch,
                                                        const uint32_t *__restrict__ push_mode, uint32_t push_stride) {
    if (push_mode && push_mode[(size_t)blockIdx.y * push_stride]) return;
    const RestrictDesc d = descs[blockIdx.y];
    const uint4 ch = dir.chunks[blockIdx.x];
    uint32_t *cp = scratch + 2ull * (d.heavy_slot + ch.x);   // {count, ticket}
    __shared__ uint32_t s_skip, s_last, s_red[8];
    if (threadIdx.x == 0) s_skip = (*(volatile uint32_t *)cp) >= d.sat;
    __syncthreads();
    uint32_t c = 0;
    if (!s_skip) {
        for (uint32_t k = ch.y + threadIdx.x; k < ch.z; k += 1024) {
            uint32_t y[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) y[u] = k + u * 256 < ch.z ? __ldg(dir.col + k + u * 256) : 0xffffffffu;
#pragma unroll
            for (int u = 0; u < 4; ++u) if (y[u] != 0xffffffffu) c += probe(d.child, y[u], d.cmask);
        }
    }
    c = __reduce_add_sync(FULL, c);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int i = 0; i < 8; ++i) tot += s_red[i];
        if (tot) atomicAdd(cp, tot);
        __threadfence();
        const uint32_t t = atomicAdd(cp + 1, 1u);
        s_last = (t == __ldg(dir.heavy_nchunks + ch.x) - 1);
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        const uint32_t tot = atomicAdd(cp, 0u);
        const uint32_t x = __ldg(dir.heavy_x + ch.x);
        if (pred_eval(d.pred, min(tot, d.sat), d.n)) {
            const uint32_t bit = 1u << (x & 31);
            if (d.out) atomicOr(d.out + (x >> 5), bit);
            if (d.proj) proj_scatter(kb, d.proj, x >> 5, bit);
            if (d.cover >= 0) {
                hedl_counts *cc = counts + d.cover;
                if (__ldg(kb.pos + (x >> 5)) & bit) {
                    atomicAdd((unsigned long long *)&cc->tp, 1ull);
                    atomicAdd((unsigned long long *)&cc->fn, ~0ull);
                }
                if (__ldg(kb.neg + (x >> 5)) & bit) {
                    atomicAdd((unsigned long long *)&cc->fp, 1ull);
                    atomicAdd((unsigned long long *)&cc->tn, ~0ull);
                }
            }
        }
        cp[0] = 0;   // self-clean: the scratch is zero again for the next launch
        cp[1] = 0;
    }
}

// ------------------------------------------------------------------------------
// Direction-optimising restriction (latency path): when the counted set
// S = child ^ cmask -- or its complement -- is sparse, walk its members y and their neighbours
// x through the inverse direction's CSR ((x, y) in rho  <=>  x in rho^-(y))
// instead of probing the child bit of every edge of every x: work |S| x mean degree instead
// of E.  Modes, decided on the device per node: 1 = push S (the flag "x has an S-neighbour"
// when the count saturates at 1, else per-x counters), 2 = push the complement of S into
// counters, cnt_S(x) = deg(x) - cnt_notS(x), 0 = the pull sweep.  Per node j of the launch:
// scratch push + j*stride words = {S count, mode, ticket} then the flag row (W4 words) and N
// u32 counters.  Both directions are launched; each node runs in exactly one (the pull
// kernels return for push nodes, the push kernels for pull nodes).  Flags and counters are
// read and zeroed by the finishing kernel, the header by k_push_reset (all zero between
// launches: another group's heavy-row counters may reuse the bytes).
__device__ __forceinline__ uint32_t *push_flags(uint32_t *base, uint32_t W4) { return base + 16; }
__device__ __forceinline__ uint32_t *push_cnts(uint32_t *base, uint32_t W4) { return base + 16 + W4; }

// |S| per node, the last block to finish picks the mode
__global__ void __launch_bounds__(256) k_push_count(KbDev kb, const RestrictDesc *__restrict__ descs, uint32_t *push,
                                                    uint32_t stride) {
    const RestrictDesc d = descs[blockIdx.y];
    uint32_t *hdr = push + (size_t)blockIdx.y * stride;
    __shared__ uint32_t s_red[8];
    uint32_t c = 0;
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < kb.W; w += gridDim.x * blockDim.x) {
        uint32_t v = __ldg(d.child + w) ^ d.cmask;
        if (w == kb.W - 1 && (kb.N & 31)) v &= (1u << (kb.N & 31)) - 1u;
        c += __popc(v);
    }
    c = __reduce_add_sync(FULL, c);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int q = 0; q < 8; ++q) t += s_red[q];
        if (t) atomicAdd(hdr, t);
        __threadfence();
        if (atomicAdd(hdr + 2, 1u) == gridDim.x - 1) {    // last block: the total is final
            __threadfence();
            const uint64_t cs = atomicAdd(hdr, 0u);
            // below N/4 members the push walks fewer edges than the pull probes, even with
            // the pull's early exit
            hdr[1] = cs * 4 <= kb.N ? 1u : ((uint64_t)kb.N - cs) * 4 <= kb.N ? 2u : 0u;
        }
    }
}

__global__ void k_push_reset(uint32_t *push, uint32_t stride, uint32_t nd) {
    const uint32_t j = threadIdx.x;
    if (j < nd) {
        uint32_t *h = push + (size_t)j * stride;
        h[0] = h[1] = h[2] = 0;
    }
}

__device__ __forceinline__ void push_edge(bool bitmode, uint32_t *flags, uint32_t *cnts, uint32_t x) {
    if (bitmode) atomicOr(flags + (x >> 5), 1u << (x & 31));
    else atomicAdd(cnts + x, 1u);
}

// light and medium members: lane per word of the pushed set, each lane walks its members'
// inverse rows (32 independent chains per warp); heavy rows are k_push_heavy's
__global__ void __launch_bounds__(256) k_push_scatter(KbDev kb, DirDev inv, const RestrictDesc *__restrict__ descs,
                                                      uint32_t *push, uint32_t stride) {
    uint32_t *hdr = push + (size_t)blockIdx.y * stride;
    const uint32_t mode = hdr[1];
    if (!mode) return;
    const RestrictDesc d = descs[blockIdx.y];
    const bool bitmode = mode == 1 && d.sat <= 1;
    const uint32_t flip = mode == 2 ? FULL : 0u;
    uint32_t *flags = push_flags(hdr, kb.W4), *cnts = push_cnts(hdr, kb.W4);
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= kb.W) return;
    uint32_t v = __ldg(d.child + w) ^ d.cmask ^ flip;
    if (w == kb.W - 1 && (kb.N & 31)) v &= (1u << (kb.N & 31)) - 1u;
    for (; v; v &= v - 1) {
        const uint32_t y = 32 * w + __ffs(v) - 1;
        const uint32_t a = __ldg(inv.row_ptr + y), b = __ldg(inv.row_ptr + y + 1);
        if (b - a > kHeavyDeg) continue;
        uint32_t e = a;
        for (; e + 4 <= b; e += 4) {                     // four neighbour ids in flight
            uint32_t x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = __ldg(inv.col + e + u);
#pragma unroll
            for (int u = 0; u < 4; ++u) push_edge(bitmode, flags, cnts, x[u]);
        }
        for (; e < b; ++e) push_edge(bitmode, flags, cnts, __ldg(inv.col + e));
    }
}

// heavy members: the inverse direction's heavy rows in 4,096-edge chunks, a CTA per chunk
__global__ void __launch_bounds__(256) k_push_heavy(KbDev kb, DirDev inv, const RestrictDesc *__restrict__ descs,
                                                    uint32_t *push, uint32_t stride) {
    uint32_t *hdr = push + (size_t)blockIdx.y * stride;
    const uint32_t mode = hdr[1];
    if (!mode) return;
    const RestrictDesc d = descs[blockIdx.y];
    const uint4 ch = inv.chunks[blockIdx.x];
    const uint32_t y = __ldg(inv.heavy_x + ch.x);
    const uint32_t in_s = (((__ldg(d.child + (y >> 5)) ^ d.cmask) >> (y & 31)) & 1u);
    if (in_s == (mode == 2 ? 1u : 0u)) return;           // y is not in the pushed set
    const bool bitmode = mode == 1 && d.sat <= 1;
    uint32_t *flags = push_flags(hdr, kb.W4), *cnts = push_cnts(hdr, kb.W4);
    for (uint32_t e = ch.y + threadIdx.x; e < ch.z; e += blockDim.x) push_edge(bitmode, flags, cnts, __ldg(inv.col + e));
}

// result words of push nodes: predicate on the flag (count saturating at 1), the counter, or
// deg - the complement's counter; tail masked; the pull kernels' epilogue (row, projection,
// coverage).  Bit mode: lane per word; counters: lane per individual, ballot per word.
__global__ void __launch_bounds__(256) k_push_finish(KbDev kb, DirDev dir, const RestrictDesc *__restrict__ descs,
                                                     uint32_t *push, uint32_t stride, hedl_counts *counts) {
    uint32_t *hdr = push + (size_t)blockIdx.y * stride;
    const uint32_t mode = hdr[1];
    if (!mode) return;
    const RestrictDesc d = descs[blockIdx.y];
    const bool bitmode = mode == 1 && d.sat <= 1;
    uint32_t *flags = push_flags(hdr, kb.W4), *cnts = push_cnts(hdr, kb.W4);
    const uint32_t lane = threadIdx.x & 31;
    uint32_t tp = 0, fp = 0;
    if (bitmode) {
        const uint32_t v1 = pred_eval(d.pred, 1u, d.n) ? FULL : 0u, v0 = pred_eval(d.pred, 0u, d.n) ? FULL : 0u;
        for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < kb.W4; w += gridDim.x * blockDim.x) {
            const uint32_t f = flags[w];
            if (f) flags[w] = 0;                          // self-clean
            uint32_t word = (f & v1) | (~f & v0);
            if (w >= kb.W) word = 0;
            else if (w == kb.W - 1 && (kb.N & 31)) word &= (1u << (kb.N & 31)) - 1u;
            if (d.out) d.out[w] = word;
            if (d.proj && w < kb.W) proj_scatter(kb, d.proj, w, word);
            if (d.cover >= 0 && w < kb.W) {
                tp += __popc(word & __ldg(kb.pos + w));
                fp += __popc(word & __ldg(kb.neg + w));
            }
        }
    } else {
        for (uint32_t w = blockIdx.x * 8 + (threadIdx.x >> 5); w < kb.W4; w += gridDim.x * 8) {
            const uint32_t x = 32 * w + lane;
            bool r = false;
            if (x < kb.N) {
                uint32_t c = cnts[x];
                if (c) cnts[x] = 0;
                if (mode == 2) c = __ldg(dir.row_ptr + x + 1) - __ldg(dir.row_ptr + x) - c;
                r = pred_eval(d.pred, min(c, d.sat), d.n);
            }
            const uint32_t word = __ballot_sync(FULL, r);
            if (lane == 0) {
                if (d.out) d.out[w] = word;
                if (d.proj && w < kb.W) proj_scatter(kb, d.proj, w, word);
                if (d.cover >= 0 && w < kb.W) {
                    tp += __popc(word & __ldg(kb.pos + w));
                    fp += __popc(word & __ldg(kb.neg + w));
                }
            }
        }
    }
    if (d.cover >= 0) block_cover(counts, d.cover, tp, fp);
}

// ------------------------------------------------------------------------------
// warp per 4 output words (lane = individual): the 4 words' row bounds and binary-search
// probes are issued together (4 independent loads in flight per lane instead of 1)
constexpr uint32_t kDrWords = 4;

// UMAP: evaluated over the U space of one direction: position p of the
// output row is the individual xmap[p]; no projection / coverage there
template <bool UMAP>
__global__ void __launch_bounds__(256) k_drange(KbDev kb, const uint32_t *__restrict__ row_ptr,
                                                const float *__restrict__ val, const DrangeDesc *__restrict__ descs,
                                                hedl_counts *counts, const uint32_t *__restrict__ xmap) {
    const DrangeDesc d = descs[blockIdx.y];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * kDrWords;
    uint32_t lo[kDrWords], hi[kDrWords], end[kDrWords];
#pragma unroll
    for (uint32_t u = 0; u < kDrWords; ++u) {
        const uint32_t pos = ((w0 + u) << 5) + lane;
        lo[u] = hi[u] = end[u] = 0;
        if (w0 + u < kb.W && pos < kb.N) {
            const uint32_t x = UMAP ? __ldg(xmap + pos) : pos;
            lo[u] = __ldg(row_ptr + x);
            hi[u] = end[u] = __ldg(row_ptr + x + 1);
        }
    }
    // first value >= d.lo in each ascending segment (interleaved binary searches)
    for (;;) {
        bool any = false;
#pragma unroll
        for (uint32_t u = 0; u < kDrWords; ++u)
            if (lo[u] < hi[u]) {
                any = true;
                const uint32_t mid = (lo[u] + hi[u]) >> 1;
                if (__ldg(val + mid) < d.lo) lo[u] = mid + 1; else hi[u] = mid;
            }
        if (!any) break;
    }
    uint32_t tp = 0, fp = 0;
#pragma unroll
    for (uint32_t u = 0; u < kDrWords; ++u) {
        const uint32_t w = w0 + u;
        const bool res = lo[u] < end[u] && __ldg(val + lo[u]) <= d.hi;
        const uint32_t word = __ballot_sync(FULL, res);
        if (lane == 0 && w < kb.W4) {
            if (!UMAP && d.proj && w < kb.W) proj_scatter(kb, d.proj, w, word);
            if (d.out) d.out[w] = word;
            if (!UMAP && d.cover >= 0 && w < kb.W) {
                tp += __popc(word & __ldg(kb.pos + w));
                fp += __popc(word & __ldg(kb.neg + w));
            }
        }
    }
    if (!UMAP && d.cover >= 0) block_cover(counts, d.cover, tp, fp);
}

// All range nodes of one data property in one pass (a launch group of k_drange nodes shares
// row_ptr / val): blockIdx.y takes kDrMulti nodes, a lane reads its individual's values once
// (up to kDrCache in registers; longer segments binary-search per node) and tests every node's
// [lo, hi]; the node words come out of ballots, lane k keeping node k's word, so the stores,
// projection scatters and coverage run one node per lane.  The values are read once per
// kDrMulti nodes instead of once per node (C5: ~43 nodes per group over 1.5·10^7 values).
constexpr uint32_t kDrMulti = 32, kDrCache = 4;
template <bool UMAP>
__global__ void __launch_bounds__(256) k_drange_multi(KbDev kb, const uint32_t *__restrict__ row_ptr,
                                                      const float *__restrict__ val, const DrangeDesc *__restrict__ descs,
                                                      uint32_t n_desc, hedl_counts *counts, const uint32_t *__restrict__ xmap) {
    __shared__ float s_lo[kDrMulti], s_hi[kDrMulti];
    __shared__ uint32_t s_tp[kDrMulti], s_fp[kDrMulti];
    const uint32_t k0 = blockIdx.y * kDrMulti, nk = min(kDrMulti, n_desc - k0);
    const uint32_t lane = threadIdx.x & 31;
    if (threadIdx.x < kDrMulti) {
        const bool v = threadIdx.x < nk;
        s_lo[threadIdx.x] = v ? descs[k0 + threadIdx.x].lo : 1.0f;    // an empty range for
        s_hi[threadIdx.x] = v ? descs[k0 + threadIdx.x].hi : 0.0f;    // the unused slots
        s_tp[threadIdx.x] = s_fp[threadIdx.x] = 0;
    }
    __syncthreads();
    DrangeDesc mine{};
    const bool has = lane < nk;
    if (has) mine = descs[k0 + lane];
    uint32_t tp = 0, fp = 0;
    const uint32_t w0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * kDrWords;
    for (uint32_t u = 0; u < kDrWords; ++u) {
        const uint32_t w = w0 + u;
        if (w >= kb.W4) break;                                       // warp-uniform
        const uint32_t pos = (w << 5) + lane;
        uint32_t a = 0, b = 0;
        if (w < kb.W && pos < kb.N) {
            const uint32_t x = UMAP ? __ldg(xmap + pos) : pos;
            a = __ldg(row_ptr + x);
            b = __ldg(row_ptr + x + 1);
        }
        float v[kDrCache];
#pragma unroll
        for (uint32_t q = 0; q < kDrCache; ++q) v[q] = a + q < b ? __ldg(val + a + q) : __int_as_float(0x7fc00000);   // NaN: no match
        const bool longseg = b - a > kDrCache;
        uint32_t word_mine = 0;
        for (uint32_t k = 0; k < nk; ++k) {
            const float lo = s_lo[k], hi = s_hi[k];
            bool hit = false;
            if (!longseg) {
#pragma unroll
                for (uint32_t q = 0; q < kDrCache; ++q) hit |= v[q] >= lo && v[q] <= hi;
            } else {                                                 // first value >= lo (sorted)
                uint32_t l = a, h = b;
                while (l < h) {
                    const uint32_t m = (l + h) >> 1;
                    if (__ldg(val + m) < lo) l = m + 1; else h = m;
                }
                hit = l < b && __ldg(val + l) <= hi;
            }
            const uint32_t word = __ballot_sync(FULL, hit);
            if (lane == k) word_mine = word;
        }
        if (has) {
            if (!UMAP && mine.proj && w < kb.W) proj_scatter(kb, mine.proj, w, word_mine);
            if (mine.out) mine.out[w] = word_mine;
            if (!UMAP && mine.cover >= 0 && w < kb.W) {
                tp += __popc(word_mine & __ldg(kb.pos + w));
                fp += __popc(word_mine & __ldg(kb.neg + w));
            }
        }
    }
    if (!UMAP && has && mine.cover >= 0 && (tp | fp)) {
        atomicAdd(&s_tp[lane], tp);
        atomicAdd(&s_fp[lane], fp);
    }
    __syncthreads();
    if (!UMAP && threadIdx.x < nk) {
        const int slot = descs[k0 + threadIdx.x].cover;
        const uint32_t a = s_tp[threadIdx.x], b = s_fp[threadIdx.x];
        if (slot >= 0) {
            hedl_counts *c = counts + slot;
            if (a) {
                atomicAdd((unsigned long long *)&c->tp, (unsigned long long)a);
                atomicAdd((unsigned long long *)&c->fn, (unsigned long long)(0ull - a));
            }
            if (b) {
                atomicAdd((unsigned long long *)&c->fp, (unsigned long long)b);
                atomicAdd((unsigned long long *)&c->tn, (unsigned long long)(0ull - b));
            }
        }
    }
}

// ------------------------------------------------------------------------------
// String restrictions (Algs. 11-14).  Pull form: lane = subject x,
// one warp per output word.  EQUAL compares interned ids (binary search of the
// subject's ascending value ids); CONTAIN tests the subject's distinct values for
// the pattern as a byte substring, lanes with many values scanned warp-cooperatively
// with the paper's early exit (stop at the first matching assertion, Alg. 13).
__device__ __forceinline__ bool str_contains(const uint8_t *__restrict__ t, uint64_t tl,
                                             const uint8_t *__restrict__ p, uint32_t pl) {
    if (pl > tl) return false;
    const uint8_t p0 = __ldg(p);
    for (uint64_t i = 0, last = tl - pl; i <= last; ++i) {
        if (__ldg(t + i) != p0) continue;
        uint32_t j = 1;
        while (j < pl && __ldg(t + i + j) == __ldg(p + j)) ++j;
        if (j == pl) return true;
    }
    return false;
}

__device__ __forceinline__ bool value_contains(const StrDev &sd, uint32_t v, const StringDesc &d) {
    const uint64_t a = __ldg(sd.dict_off + v), b = __ldg(sd.dict_off + v + 1);
    return str_contains(sd.dict + a, b - a, d.pat, d.pat_len);
}

constexpr uint32_t kStrLaneDeg = 8;   // CONTAIN rows longer than this are scanned by the whole warp

__global__ void __launch_bounds__(256) k_string(KbDev kb, StrDev sd, const StringDesc *__restrict__ descs,
                                                hedl_counts *counts) {
    const StringDesc d = descs[blockIdx.y];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * kDrWords;   // 4 words per warp
    uint32_t e0[kDrWords], e1[kDrWords];
#pragma unroll
    for (uint32_t u = 0; u < kDrWords; ++u) {
        const uint32_t x = ((w0 + u) << 5) + lane;
        e0[u] = e1[u] = 0;
        if (w0 + u < kb.W && x < kb.N) {
            e0[u] = __ldg(sd.row_ptr + x);
            e1[u] = __ldg(sd.row_ptr + x + 1);
        }
    }
    uint32_t words[kDrWords];
    if (d.mode == SM_EQUAL) {
        uint32_t lo[kDrWords], hi[kDrWords];
#pragma unroll
        for (uint32_t u = 0; u < kDrWords; ++u) { lo[u] = e0[u]; hi[u] = e1[u]; }
        for (;;) {                                          // first id >= vid, searches interleaved
            bool any = false;
#pragma unroll
            for (uint32_t u = 0; u < kDrWords; ++u)
                if (lo[u] < hi[u]) {
                    any = true;
                    const uint32_t mid = (lo[u] + hi[u]) >> 1;
                    if (__ldg(sd.vid + mid) < d.vid) lo[u] = mid + 1; else hi[u] = mid;
                }
            if (!any) break;
        }
#pragma unroll
        for (uint32_t u = 0; u < kDrWords; ++u)
            words[u] = __ballot_sync(FULL, lo[u] < e1[u] && __ldg(sd.vid + lo[u]) == d.vid);
    } else {
#pragma unroll
        for (uint32_t u = 0; u < kDrWords; ++u) {
            bool res = false;
            const bool longrow = e1[u] - e0[u] > kStrLaneDeg;
            if (!longrow)
                for (uint32_t e = e0[u]; e < e1[u] && !res; ++e) res = value_contains(sd, __ldg(sd.vid + e), d);
            uint32_t word = __ballot_sync(FULL, res);
            for (uint32_t m = __ballot_sync(FULL, longrow); m; m &= m - 1) {
                const uint32_t L = __ffs(m) - 1;
                const uint32_t a = __shfl_sync(FULL, e0[u], L), b = __shfl_sync(FULL, e1[u], L);
                for (uint32_t base = a; base < b; base += 32) {          // uniform trip count
                    const uint32_t e = base + lane;
                    const bool hit = e < b && value_contains(sd, __ldg(sd.vid + e), d);
                    if (__any_sync(FULL, hit)) { word |= 1u << L; break; }
                }
            }
            words[u] = word;
        }
    }
    uint32_t tp = 0, fp = 0;
#pragma unroll
    for (uint32_t u = 0; u < kDrWords; ++u) {
        const uint32_t w = w0 + u;
        if (lane == 0 && w < kb.W4) {
            if (d.proj && w < kb.W) proj_scatter(kb, d.proj, w, words[u]);
            if (d.out) d.out[w] = words[u];
            if (d.cover >= 0 && w < kb.W) {
                tp += __popc(words[u] & __ldg(kb.pos + w));
                fp += __popc(words[u] & __ldg(kb.neg + w));
            }
        }
    }
    if (d.cover >= 0) block_cover(counts, d.cover, tp, fp);
}

__global__ void k_gather_counts(const hedl_counts *__restrict__ slots, const uint32_t *__restrict__ slot_of,
                                hedl_counts *out, uint32_t n) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = slots[slot_of[i]];
}

__global__ void k_gather_bits(const uint32_t *const *__restrict__ rows, uint32_t *out, uint32_t W) {
    const uint32_t *src = rows[blockIdx.y];
    uint32_t *dst = out + (uint64_t)blockIdx.y * W;
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x) dst[w] = src[w];
}
}  // namespace

// ---- launchers -------------------------------------------------------------------
static inline uint32_t cdiv(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }

void launch_cover_init(cudaStream_t s, hedl_counts *counts, uint32_t n, uint64_t npos, uint64_t nneg) {
    if (!n) return;
    prof_begin(s, KC_COVER_INIT);
    k_cover_init<<<cdiv(n, 256), 256, 0, s>>>(counts, n, npos, nneg);
    count_launch();
    prof_end(s, KC_COVER_INIT, 32.0 * n, n);
}

// full_rows: the rows span all N individuals (HBM-sized); otherwise they are example-projected
// or U rows (kilobytes per row, L2-resident) and the launch is profiled as its own class
void launch_bool(cudaStream_t s, const KbDev &kb, const BoolDesc *d_desc, uint32_t n_desc,
                 const Operand *d_ops, hedl_counts *counts, double alg_bytes, uint64_t npos, uint64_t nneg,
                 bool full_rows) {
    const int kc = full_rows ? KC_BOOL : KC_BOOL_L2;
    // a warp per node unless the launch has too few nodes to fill the SMs with warps while its
    // rows are long (a few hundred U-space fillers of 5,000-word rows: one warp walking a row
    // is a chain of ~20 dependent loads) -- then a CTA per row chunk (k_bool)
    const bool few_long = n_desc < 148u * 8u && (kb.W4 >> 2) >= 256;
    if (kb.W4 && (kb.W4 >> 2) <= kBoolWarpMaxN4 && n_desc >= 64 && !few_long) {
        const uint32_t g = std::min<uint32_t>(cdiv(n_desc, 8), 148u * 16u);
        prof_begin(s, kc);
        if (full_rows) k_bool_warp<true><<<g, 256, 0, s>>>(kb, d_desc, n_desc, d_ops, counts, npos, nneg);
        else k_bool_warp<false><<<g, 256, 0, s>>>(kb, d_desc, n_desc, d_ops, counts, npos, nneg);
        count_launch();
        prof_end(s, kc, alg_bytes, n_desc);
        return;
    }
    for (uint32_t off = 0; off < n_desc; off += 65535) {
        const uint32_t nd = n_desc - off < 65535 ? n_desc - off : 65535;
        const uint32_t g1 = kb.W4 ? cdiv(kb.W4 / 4, 256) : 0;         // one uint4 per thread
        if (!g1) return;
        const uint32_t gU = cdiv(kb.W4 / 4, 256 * kBoolU);              // kBoolU per thread
        // kBoolU words per thread when the launch has enough nodes to fill the 148 SMs,
        // more CTAs per node (down to one word per thread) when it has few
        const uint32_t want = std::max<uint32_t>(gU, std::min<uint32_t>(g1, cdiv(148u * 8u, nd)));
        dim3 grid(want, nd);
        prof_begin(s, kc);
        if (full_rows) k_bool<true><<<grid, 256, 0, s>>>(kb, d_desc + off, d_ops, counts);
        else k_bool<false><<<grid, 256, 0, s>>>(kb, d_desc + off, d_ops, counts);
        count_launch();
        prof_end(s, kc, alg_bytes * nd / n_desc, nd);
    }
}

size_t push_scratch_words(uint32_t N, uint32_t W4, bool counting) {
    return (size_t)16 + W4 + (counting ? (size_t)N : 0) + 16;
}

void launch_restrict(cudaStream_t s, const KbDev &kb, const DirDev &dir, const RestrictDesc *d_desc,
                     uint32_t n_desc, hedl_counts *counts, uint32_t *heavy_scratch, double alg_light,
                     double alg_heavy, const DirDev *inv, uint32_t *push, size_t push_stride) {
    const uint32_t gx = dir.n_tiles;
    if (!gx || !kb.W4) return;
    const bool use_push = inv && push && n_desc <= kPushMaxNodes;
    if (use_push) {
        // direction decision on the device: |S| per node, then each node runs push or pull
        const uint32_t stride = (uint32_t)push_stride;
        // (the headers are zero: k_push_reset cleans them after every launch)
        prof_begin(s, KC_RESTRICT);
        k_push_count<<<dim3(std::min<uint32_t>(cdiv(kb.W, 256), 148u * 4u), n_desc), 256, 0, s>>>(kb, d_desc, push, stride);
        k_push_scatter<<<dim3(cdiv(kb.W, 256), n_desc), 256, 0, s>>>(kb, *inv, d_desc, push, stride);
        if (inv->n_chunks) k_push_heavy<<<dim3(inv->n_chunks, n_desc), 256, 0, s>>>(kb, *inv, d_desc, push, stride);
        k_push_finish<<<dim3(std::min<uint32_t>(cdiv(kb.W4, 256), 148u * 8u), n_desc), 256, 0, s>>>(kb, dir, d_desc, push,
                                                                                                 stride, counts);
        for (int q = 0; q < 4; ++q) count_launch();
        prof_end(s, KC_RESTRICT, 0, n_desc);
    }
    const uint32_t *pm = use_push ? push + 1 : nullptr;
    for (uint32_t off = 0; off < n_desc; off += 65535) {
        const uint32_t nd = n_desc - off < 65535 ? n_desc - off : 65535;
        prof_begin(s, KC_RESTRICT);
        k_restrict_tile<<<dim3(gx, nd), 256, 0, s>>>(kb, dir, d_desc + off, counts, pm, (uint32_t)push_stride);
        count_launch();
        prof_end(s, KC_RESTRICT, alg_light * nd / n_desc, nd);
        if (dir.n_chunks) {
            prof_begin(s, KC_HEAVY);
            k_restrict_heavy<<<dim3(dir.n_chunks, nd), 256, 0, s>>>(kb, dir, d_desc + off, counts, heavy_scratch, pm,
                                                                    (uint32_t)push_stride);
            count_launch();
            prof_end(s, KC_HEAVY, alg_heavy * nd / n_desc, nd);
        }
    }
    if (use_push) {
        k_push_reset<<<1, 32, 0, s>>>(push, (uint32_t)push_stride, n_desc);
        count_launch();
    }
}

void launch_drange(cudaStream_t s, const KbDev &kb, const uint32_t *row_ptr, const float *val,
                   const DrangeDesc *d_desc, uint32_t n_desc, hedl_counts *counts, double alg_bytes,
                   const uint32_t *xmap) {
    const uint32_t gx = cdiv(kb.W4, 8 * kDrWords);
    if (!gx) return;
    static const bool no_multi = std::getenv("HEDL_NO_DRANGE_MULTI") != nullptr;
    if (n_desc >= 2 && !no_multi) {                 // one pass over the values for every node
        for (uint32_t off = 0; off < n_desc; off += 65535u * kDrMulti) {
            const uint32_t nd = std::min<uint32_t>(n_desc - off, 65535u * kDrMulti);
            prof_begin(s, KC_DRANGE);
            if (xmap) k_drange_multi<true><<<dim3(gx, cdiv(nd, kDrMulti)), 256, 0, s>>>(kb, row_ptr, val, d_desc + off, nd, counts, xmap);
            else k_drange_multi<false><<<dim3(gx, cdiv(nd, kDrMulti)), 256, 0, s>>>(kb, row_ptr, val, d_desc + off, nd, counts, nullptr);
            count_launch();
            // the segment arrays once per kDrMulti nodes (the per-node model's share) + the rows
            prof_end(s, KC_DRANGE, alg_bytes / n_desc * cdiv(nd, kDrMulti) + 4.0 * kb.W * nd, nd);
        }
        return;
    }
    for (uint32_t off = 0; off < n_desc; off += 65535) {
        const uint32_t nd = n_desc - off < 65535 ? n_desc - off : 65535;
        prof_begin(s, KC_DRANGE);
        if (xmap) k_drange<true><<<dim3(gx, nd), 256, 0, s>>>(kb, row_ptr, val, d_desc + off, counts, xmap);
        else k_drange<false><<<dim3(gx, nd), 256, 0, s>>>(kb, row_ptr, val, d_desc + off, counts, nullptr);
        count_launch();
        prof_end(s, KC_DRANGE, alg_bytes * nd / n_desc, nd);
    }
}

void launch_string(cudaStream_t s, const KbDev &kb, const StrDev &sd, const StringDesc *d_desc, uint32_t n_desc,
                   hedl_counts *counts, double alg_bytes) {
    const uint32_t gx = cdiv(kb.W4, 8 * kDrWords);
    if (!gx) return;
    for (uint32_t off = 0; off < n_desc; off += 65535) {
        const uint32_t nd = n_desc - off < 65535 ? n_desc - off : 65535;
        prof_begin(s, KC_STRING);
        k_string<<<dim3(gx, nd), 256, 0, s>>>(kb, sd, d_desc + off, counts);
        count_launch();
        prof_end(s, KC_STRING, alg_bytes * nd / n_desc, nd);
    }
}

void launch_gather_counts(cudaStream_t s, const hedl_counts *slots, const uint32_t *slot_of,
                          hedl_counts *out, uint32_t n) {
    if (!n) return;
    prof_begin(s, KC_GATHER);
    k_gather_counts<<<cdiv(n, 256), 256, 0, s>>>(slots, slot_of, out, n);
    count_launch();
    prof_end(s, KC_GATHER, 68.0 * n, n);
}

void launch_gather_bits(cudaStream_t s, const uint32_t *const *rows, uint32_t *out, uint32_t W, uint32_t n) {
    if (!n || !W) return;
    for (uint32_t off = 0; off < n; off += 65535) {
        const uint32_t nd = n - off < 65535 ? n - off : 65535;
        prof_begin(s, KC_GATHER);
        // about 16 CTAs per SM over all rows of the launch, each thread ~4 words (one 10^7-bit
        // row is 1.25 MB: 32 CTAs per row took 18 us)
        const uint32_t gx = std::max<uint32_t>(1, std::min<uint32_t>(cdiv(W, 1024), cdiv(2368, nd)));
        k_gather_bits<<<dim3(gx, nd), 256, 0, s>>>(rows + off, out + (uint64_t)off * W, W);
        count_launch();
        prof_end(s, KC_GATHER, 8.0 * W * nd, nd);
    }
}

}  // namespace hedl

// Lane-packed ("bit-sliced") batch restriction kernels (SURVEY 8(d) "Optional
// bit-sliced batch variant").
//
// Up to 256 restriction nodes on one role direction form a pack: lane j of the
// pack is node j.  One CSR pass then evaluates all 256 nodes:
//   k_slice_pack   T[y] = 256-bit word of child_j(y) ^ cmask_j   (32x32 warp bit transposes)
//   k_slice_heavy  heavy rows (deg > kHeavyDeg) in CTA chunks, combined with atomics
//   k_slice_tile   per 1024-individual tile: for every x, acc = OR / saturating count of
//                  T[y] over y in N(x) (thread per light row, warp per medium row), the
//                  per-lane predicate, then transpose back to the nodes' bitset rows with
//                  fused Alg. 15 coverage.
// OR packs hold nodes whose count saturates at 1 (exists, forall, >=1, <=0, ...);
// COUNT packs keep 5-plane bit-sliced saturating counters (counts 0..31, n <= 30).
// Semantics are exactly the per-node kernels' (kernels.cu): same predicates,
// same saturation rule (pred(min(cnt, sat)) == pred(cnt)).
#include "slice.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace hedl {

namespace {
constexpr uint32_t FULL = 0xffffffffu;
constexpr int LW = 8;             // u32 words per individual in T: 256 lanes
constexpr int NPL = 5;            // counter bit planes (0..31)
constexpr int TROW = LW + 1;      // smem row stride (bank-conflict-free transposes)

struct SliceDir {
    const uint32_t *row_ptr, *col;
    const uint4 *tiles;           // [n_tiles + 1] {order begin, n_med, n_light, heavy begin}
    const uint32_t *order;
    const uint32_t *tile_rank;    // [n_tiles] tiles in decreasing sweep cost
    const uint32_t *tile_nbig;    // [n_tiles] medium rows with deg > kMidDeg (the first of the tile's medium rows)
    const uint32_t *tile_slice, *sell_off, *sell_w, *sell_col;   // SELL-16 light rows
    const uint32_t *heavy_x, *heavy_nchunks;
    const uint4 *chunks;
    uint32_t n_heavy, n_chunks, n_tiles;
};

// per-direction U masks for the restriction U-row epilogue (directions < kMaxUDirs)
struct UTab {
    const uint32_t *um[kMaxUDirs], *ub[kMaxUDirs];   // ex_umask / ex_ubase of direction d
    const uint32_t *ul[kMaxUDirs];                    // ulist of direction d (U position -> individual)
    uint32_t nu[kMaxUDirs];                           // |U_d|
    uint32_t stride;                                  // words between a node's consecutive U rows
};


struct SliceScratch {
    uint4 *T;                     // [W4*32][2] : 32 B per individual
    uint32_t *hacc;               // [n_heavy][8]     OR accumulators
    uint32_t *hcnt;               // [n_heavy][256]   per-lane counts
    uint32_t *ticket;             // [n_heavy]
    uint32_t *hout;               // [n_heavy][8]     finished heavy rows
    uint64_t t_stride;            // uint4 between the T of consecutive packs of one launch
    uint64_t h_stride;            // heavy rows between the accumulators of consecutive packs
    uint64_t t_cap;               // uint4 of one pack's T region (HCHECK bound of the gathers)
    __device__ __forceinline__ SliceScratch at(uint32_t p) const {
        SliceScratch r = *this;
        r.T += p * t_stride;
        r.hacc += p * h_stride * 8;
        r.hcnt += p * h_stride * 256;
        r.ticket += p * h_stride;
        r.hout += p * h_stride * 8;
        return r;
    }
};

// pack p of a run of consecutive same-class descriptors: descs [256p, min(256p + 256, run))
__device__ __forceinline__ uint32_t pack_count(uint32_t run, uint32_t p) { return min(256u, run - 256u * p); }

// per-pack lane constants, built in shared memory from the node descriptors; NP packs of one
// pass: word kk of the 8*NP covers lanes 32kk .. 32kk+31
template <int NP>
struct PackConstN {
    uint32_t fl[NP * LW], am[NP * LW], om[NP * LW];   // OR class: out = ((acc ^ fl) & am) | om
    uint32_t nb[NPL][NP * LW];                         // COUNT class: bit planes of n
    uint32_t mge[NP * LW], mle[NP * LW], meq[NP * LW], mlep[NP * LW];
};
using PackConst = PackConstN<1>;

// 32x32 bit transpose across a warp: in lane r bit c = M[r][c]; out lane c bit r = M[r][c].
// Five butterfly stages; each lane keeps half of its word and takes the other half from its
// partner.  The 16- and 8-bit stages are one byte permute (selector chosen per lane), the
// 4/2/1-bit stages one rotate (left by j for the lower lane of a pair, right by j for the
// upper one) and one LOP3 -- 13 instructions with the shuffles instead of ~30.
__device__ __forceinline__ uint32_t warp_transpose(uint32_t x, uint32_t lane) {
    const bool lo16 = !(lane & 16), lo8 = !(lane & 8), lo4 = !(lane & 4), lo2 = !(lane & 2), lo1 = !(lane & 1);
    uint32_t y = __shfl_xor_sync(FULL, x, 16);
    x = __byte_perm(x, y, lo16 ? 0x5410u : 0x3276u);
    y = __shfl_xor_sync(FULL, x, 8);
    x = __byte_perm(x, y, lo8 ? 0x6240u : 0x3715u);
    uint32_t k;
    y = __shfl_xor_sync(FULL, x, 4);
    k = lo4 ? 0x0F0F0F0Fu : 0xF0F0F0F0u;
    x = (x & k) | (__funnelshift_l(y, y, lo4 ? 4 : 28) & ~k);
    y = __shfl_xor_sync(FULL, x, 2);
    k = lo2 ? 0x33333333u : 0xCCCCCCCCu;
    x = (x & k) | (__funnelshift_l(y, y, lo2 ? 2 : 30) & ~k);
    y = __shfl_xor_sync(FULL, x, 1);
    k = lo1 ? 0x55555555u : 0xAAAAAAAAu;
    x = (x & k) | (__funnelshift_l(y, y, lo1 ? 1 : 31) & ~k);
    return x;
}

// The bits of `word` selected by `m` (pext), destined for bit positions base .. of a packed
// row (a projected or U row), gathered per destination word: one write per word touched.
// (pw, pbits) is the caller's pending destination word; flush with pack_flush at the end.
// Destination words in [own_lo, own_hi) receive bits from this caller only: a plain store;
// the others (shared with a neighbouring tile) an atomicOr into the zeroed row.
__device__ __forceinline__ void pack_flush(uint32_t *row, uint32_t pw, uint32_t pbits, uint32_t own_lo, uint32_t own_hi) {
    if (pw >= own_lo && pw < own_hi) row[pw] = pbits;
    else if (pbits) atomicOr(row + pw, pbits);
}
__device__ __forceinline__ void pack_bits(uint32_t m, uint32_t word, uint32_t base, uint32_t *row, uint32_t &pw,
                                          uint32_t &pbits, uint32_t own_lo = 0, uint32_t own_hi = 0) {
    if (!m || !word) return;
    uint32_t bits = 0, nb = 0;
    for (; m; m &= m - 1, ++nb) bits |= ((word >> (__ffs(m) - 1)) & 1u) << nb;
    if (!bits) return;                    // (words never written stay 0: the row was zeroed)
    const uint32_t wi = base >> 5, sh = base & 31;
    if (wi != pw) {
        if (pbits) pack_flush(row, pw, pbits, own_lo, own_hi);
        pw = wi;
        pbits = 0;
    }
    pbits |= bits << sh;
    if (sh + nb > 32) {
        pack_flush(row, pw, pbits, own_lo, own_hi);
        pw = wi + 1;
        pbits = bits >> (32 - sh);
    }
}

// every thread of the CTA calls; lanes >= count get "always 0" (am = om = 0, masks 0).
// Warp k builds the words of lanes 32k..32k+31 with ballots (no shared-memory atomics).
template <int NP>
__device__ void build_consts(PackConstN<NP> &pc, const RestrictDesc *__restrict__ d, uint32_t count) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t k = threadIdx.x >> 5; k < NP * LW; k += blockDim.x >> 5) {
        const uint32_t j = k * 32 + lane;
        uint32_t pred = 0xffu, n = 0;
        if (j < count) {
            pred = d[j].pred;
            n = d[j].n;
        }
        // OR class (sat <= 1): result is a function of b = (cnt >= 1)
        //   GE 0 -> 1 ; GE 1 -> b ; LE 0 / EQ 0 -> !b ; LEP 0 -> 0
        const bool ge = pred == P_GE, le = pred == P_LE, eq = pred == P_EQ, lep = pred == P_LEP;
        const uint32_t am = __ballot_sync(FULL, (ge && n != 0) || le || eq);
        const uint32_t fl = __ballot_sync(FULL, le || eq);
        const uint32_t om = __ballot_sync(FULL, ge && n == 0);
        const uint32_t mge = __ballot_sync(FULL, ge), mle = __ballot_sync(FULL, le);
        const uint32_t meq = __ballot_sync(FULL, eq), mlep = __ballot_sync(FULL, lep);
        uint32_t nb[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) nb[q] = __ballot_sync(FULL, (n >> q) & 1u);
        if (lane == 0) {
            pc.am[k] = am; pc.fl[k] = fl; pc.om[k] = om;
            pc.mge[k] = mge; pc.mle[k] = mle; pc.meq[k] = meq; pc.mlep[k] = mlep;
#pragma unroll
            for (int q = 0; q < NPL; ++q) pc.nb[q][k] = nb[q];
        }
    }
    __syncthreads();
}

// A thread owns HW = 4 words (128 lanes) of a row: the two threads of an
// adjacent lane pair (lane & 1 = half) cover the 256 lanes and gather the two
// 16 B halves of one 32 B sector of T[y] with one warp instruction.
constexpr int HW = 4;

// COUNT accumulators are 5 bit planes (count mod 32) plus a sticky overflow plane (count
// >= 32 seen); fold() saturates the planes to 31 where it is set, so every predicate
// sees min(cnt, 31) -- exact for n <= 30 (pred(min(cnt, sat)) == pred(cnt)).
template <bool COUNT>
struct Acc {
    uint32_t c[COUNT ? NPL : 1][HW];
    uint32_t ov[COUNT ? HW : 1];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int q = 0; q < (COUNT ? NPL : 1); ++q)
#pragma unroll
            for (int k = 0; k < HW; ++k) c[q][k] = 0;
#pragma unroll
        for (int k = 0; k < (COUNT ? HW : 1); ++k) ov[k] = 0;
    }
    __device__ __forceinline__ void add1(int k, uint32_t v) {
        if (!COUNT) {
            c[0][k] |= v;
        } else {
            uint32_t carry = v;                  // half-adder ripple, carry out -> overflow
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const uint32_t t = c[q][k] & carry;
                c[q][k] ^= carry;
                carry = t;
            }
            ov[k & (COUNT ? HW - 1 : 0)] |= carry;
        }
    }
    __device__ __forceinline__ void add(const uint4 v) { add1(0, v.x); add1(1, v.y); add1(2, v.z); add1(3, v.w); }
    // four inputs per word with a carry-save tree: two full adders at weight 1, one at
    // weight 2, then a half-adder ripple (13 LOP3-class ops per word instead of ~50)
    __device__ __forceinline__ void add4w(int k, uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
        if (!COUNT) {
            c[0][k] |= v0 | v1 | v2 | v3;
        } else {
            uint32_t s0 = c[0][k];
            const uint32_t k1a = (s0 & v0) | (s0 & v1) | (v0 & v1);
            s0 ^= v0 ^ v1;
            const uint32_t k1b = (s0 & v2) | (s0 & v3) | (v2 & v3);
            c[0][k] = s0 ^ v2 ^ v3;
            const uint32_t s1 = c[1][k];
            uint32_t carry = (s1 & k1a) | (s1 & k1b) | (k1a & k1b);
            c[1][k] = s1 ^ k1a ^ k1b;
#pragma unroll
            for (int q = 2; q < NPL; ++q) {
                const uint32_t t = c[q][k] & carry;
                c[q][k] ^= carry;
                carry = t;
            }
            ov[k & (COUNT ? HW - 1 : 0)] |= carry;
        }
    }
    __device__ __forceinline__ void add4(const uint4 a, const uint4 b, const uint4 c4, const uint4 d) {
        add4w(0, a.x, b.x, c4.x, d.x);
        add4w(1, a.y, b.y, c4.y, d.y);
        add4w(2, a.z, b.z, c4.z, d.z);
        add4w(3, a.w, b.w, c4.w, d.w);
    }
    // saturate the planes where the overflow plane is set (planes then hold min(cnt, 31))
    __device__ __forceinline__ void fold() {
        if (COUNT) {
#pragma unroll
            for (int k = 0; k < HW; ++k) {
#pragma unroll
                for (int q = 0; q < NPL; ++q) c[q][k] |= ov[k & (COUNT ? HW - 1 : 0)];
                ov[k & (COUNT ? HW - 1 : 0)] = 0;
            }
        }
    }
    // saturating add of another (folded) accumulator (bit-sliced ripple-carry adder)
    __device__ __forceinline__ void merge(const Acc &o) {
#pragma unroll
        for (int k = 0; k < HW; ++k) {
            if (!COUNT) {
                c[0][k] |= o.c[0][k];
            } else {
                uint32_t carry = 0;
#pragma unroll
                for (int q = 0; q < NPL; ++q) {
                    const uint32_t a = c[q][k], b = o.c[q][k];
                    c[q][k] = a ^ b ^ carry;
                    carry = (a & b) | (carry & (a ^ b));
                }
#pragma unroll
                for (int q = 0; q < NPL; ++q) c[q][k] |= carry;
            }
        }
    }
    // combine the lane groups of G lanes (G = 2: pairs, 4: quads) of an aligned block of 2*TOP
    // lanes (lanes equal mod G); every lane gets its group position's total.  TOP = 16: the
    // whole warp.
    template <int TOP = 16, int G = 2>
    __device__ __forceinline__ void warp_reduce_pairs() {
        fold();
#pragma unroll
        for (int off = TOP; off >= G; off >>= 1) {
            Acc o;
#pragma unroll
            for (int q = 0; q < (COUNT ? NPL : 1); ++q)
#pragma unroll
                for (int k = 0; k < HW; ++k) o.c[q][k] = __shfl_xor_sync(FULL, c[q][k], off);
            merge(o);
        }
    }
    template <class PC>
    __device__ __forceinline__ uint32_t result(const PC &pc, int kk, int k) const {
        if (!COUNT) return ((c[0][k] ^ pc.fl[kk]) & pc.am[kk]) | pc.om[kk];
        const uint32_t o = ov[k & (COUNT ? HW - 1 : 0)];
        uint32_t gt = 0, eq = FULL, nz = 0;
#pragma unroll
        for (int q = NPL - 1; q >= 0; --q) {
            const uint32_t cq = c[q][k] | o, nq = pc.nb[q][kk];
            gt |= eq & cq & ~nq;
            eq &= ~(cq ^ nq);
            nz |= cq;
        }
        const uint32_t ge = gt | eq, le = ~gt;
        return (ge & pc.mge[kk]) | (le & pc.mle[kk]) | (eq & pc.meq[kk]) | (le & nz & pc.mlep[kk]);
    }
};

// acc += T[y] (this thread's 16 B of the R x 16 B record, `half` = its index) for the edges
// [e, b) with stride `step`, 4 gathers in flight
template <bool COUNT, int R = 2>
__device__ __forceinline__ void scan_edges(Acc<COUNT> &acc, const uint32_t *__restrict__ col, const uint4 *__restrict__ T,
                                           uint32_t e, uint32_t b, uint32_t step, uint32_t half, uint64_t cap) {
    // software-pipelined: the next four neighbour ids are in flight during this step's gathers
    uint32_t y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) y[u] = e + step * u < b ? __ldg(col + e + step * u) : 0xffffffffu;
    for (; e < b; e += 4 * step) {
        uint32_t yn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) yn[u] = e + step * (4 + u) < b ? __ldg(col + e + step * (4 + u)) : 0xffffffffu;
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            HCHECK(y[u] == 0xffffffffu || (uint64_t)R * y[u] + R <= cap);
            v[u] = y[u] != 0xffffffffu ? __ldg(T + (uint64_t)R * y[u] + half) : make_uint4(0, 0, 0, 0);
        }
        acc.add4(v[0], v[1], v[2], v[3]);
#pragma unroll
        for (int u = 0; u < 4; ++u) y[u] = yn[u];
    }
}

// ------------------------------------------------------------------------------
// T[y] for the packs of a run (blockIdx.y = pack): a CTA stages 256 child rows x 64
// words (2048 individuals) in shared memory with one TMA bulk copy per row
// (cp.async.bulk, completion counted on an mbarrier), then warps transpose 32x32 bit
// blocks (complement masks applied on the way) and write each individual's 32 B of T.
constexpr uint32_t PK_WORDS = 32, PK_STRIDE = 36;        // 144 B rows: 16 B aligned for TMA, conflict-free quads
constexpr uint32_t PK_WPW = PK_WORDS / 8;                 // words per warp

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(256, 4) k_slice_pack(KbDev kb, const RestrictDesc *__restrict__ d_run, uint32_t run,
                                                    uint4 *__restrict__ T_base, uint64_t t_stride,
                                                    const uint32_t *__restrict__ umask, const uint32_t *__restrict__ ubase,
                                                    const Operand *__restrict__ ops, uint32_t rec) {
    extern __shared__ __align__(16) uint32_t sm[];        // [256][PK_STRIDE] lane rows
    __shared__ uint32_t s_cm[256], s_on[256];
    __shared__ uint64_t s_optab[256 * kFuseMaxOps];       // fused lanes' operand rows | complement
    __shared__ __align__(8) uint64_t mbar;
    const uint32_t p = blockIdx.y;
    const RestrictDesc *d = d_run + 256u * p;
    const uint32_t count = pack_count(run, p);
    // rec = uint4 per individual: 2 (one pack's 32 B T per region of t_stride uint4), 4 (a pack
    // pair: the two packs' 32 B interleaved in one 64 B record;
    // t_stride = the whole region) or 1 (a narrow pack of <= 128 nodes: lanes 0..127, 16 B)
    uint4 *T = rec == 4 ? T_base + 2 * p : T_base + p * t_stride;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t w0 = blockIdx.x * PK_WORDS;
    const uint32_t nwords = min(PK_WORDS, kb.W4 - w0);    // multiple of 4 (W4 and w0 are)
    const uint32_t seg = nwords * 4;
    const uint32_t mb = smem_u32(&mbar);
    const uint32_t t = threadIdx.x;
    // lane t: a materialised filler row (one TMA bulk copy of its segment) or a fused boolean
    // filler (the CTA combines the operand segments itself)
    const uint32_t *child = t < count ? d[t].child : nullptr;
    const bool tma = child != nullptr;
    const uint32_t ntma = __syncthreads_count(tma);
    const bool any_fused = ntma < min(count, 256u);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(seg * ntma) : "memory");
    }
    s_cm[t] = t < count ? d[t].cmask : 0u;
    if (t >= count)
        for (uint32_t i = 0; i < PK_WORDS; ++i) sm[t * PK_STRIDE + i] = 0u;
    if (any_fused) {
        // lane t's operand rows (32 B aligned) with the complement flag in bit 0; all descriptor
        // loads independent, so the combine has no dependent load per operand
        const uint32_t on_t = (t < count && !tma) ? d[t].op_n : 0u;
        s_on[t] = on_t;
        if (on_t) {
            const Operand *op = ops + d[t].op_first;
            const uint32_t n_t = min(on_t & 0x7fffffffu, kFuseMaxOps);
#pragma unroll
            for (uint32_t j = 0; j < kFuseMaxOps; ++j)
                if (j < n_t) {
                    const Operand o = op[j];
                    s_optab[t * kFuseMaxOps + j] = reinterpret_cast<uint64_t>(o.ptr) | (o.mask & 1u);
                }
        }
    }
    __syncthreads();                                      // barrier initialised and armed
    if (tma)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sm + t * PK_STRIDE)), "l"(child + w0), "r"(seg), "r"(mb) : "memory");
    if (any_fused) {
        // fused fillers, CTA-cooperative while the bulk copies fly: a lane's 32-word segment is 8 quads, thread t takes quad
        // t & 7 of lanes (t >> 3) + 32 r (128 contiguous bytes per lane and operand, coalesced /
        // conflict-free).  k-ary AND / OR with complement masks as in k_bool: an AND is the
        // complemented OR of the complements, one LOP3 per operand word.
        const uint32_t wq = 4 * (t & 7);
        const uint32_t lim = kb.W > w0 ? kb.W - w0 : 0u;       // valid words of this segment
        const uint32_t tail = (kb.N & 31) ? (1u << (kb.N & 31)) - 1u : FULL;
#pragma unroll
        for (uint32_t half = 0; half < 2; ++half) {
            uint32_t on[4], flip[4];
            uint4 acc[4];
            uint32_t jmax = 0;
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r) {
                const uint32_t L = (t >> 3) + 32 * (4 * half + r);
                on[r] = min(s_on[L] & 0x7fffffffu, kFuseMaxOps);
                flip[r] = (s_on[L] >> 31) ? 0u : FULL;
                acc[r] = make_uint4(0, 0, 0, 0);
                jmax = max(jmax, on[r]);
            }
            if (wq >= nwords) jmax = 0;
            for (uint32_t jo = 0; jo < jmax; ++jo) {
#pragma unroll
                for (uint32_t r = 0; r < 4; ++r) {
                    if (jo < on[r]) {
                        const uint32_t L = (t >> 3) + 32 * (4 * half + r);
                        const uint64_t e = s_optab[L * kFuseMaxOps + jo];
                        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(e & ~uint64_t(1)) + ((w0 + wq) >> 2));
                        const uint32_t m = ((e & 1u) ? FULL : 0u) ^ flip[r];
                        acc[r].x |= v.x ^ m; acc[r].y |= v.y ^ m; acc[r].z |= v.z ^ m; acc[r].w |= v.w ^ m;
                    }
                }
            }
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r) {
                if (!on[r] || wq >= nwords) continue;
                const uint32_t L = (t >> 3) + 32 * (4 * half + r);
                uint32_t v4[4] = {acc[r].x ^ flip[r], acc[r].y ^ flip[r], acc[r].z ^ flip[r], acc[r].w ^ flip[r]};
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k) {       // tail bits (>= N) and padding words stay 0
                    const uint32_t wl = wq + k;
                    if (wl >= lim) v4[k] = 0u;
                    else if (w0 + wl + 1 == kb.W) v4[k] &= tail;
                }
                *reinterpret_cast<uint4 *>(sm + L * PK_STRIDE + wq) = make_uint4(v4[0], v4[1], v4[2], v4[3]);
            }
        }
    }
    // EX packs: T only at the example rows' neighbours U, compacted (umask / ubase); the
    // masks of this warp's PK_WPW words are fetched while the bulk copies are in flight
    uint32_t ums[PK_WPW], ubs[PK_WPW];
#pragma unroll
    for (uint32_t k = 0; k < PK_WPW; ++k) {
        const uint32_t w = w0 + wid * PK_WPW + k;
        ums[k] = (umask && w < kb.W4) ? __ldg(umask + w) : FULL;
        ubs[k] = (umask && w < kb.W4) ? __ldg(ubase + w) : 0u;
    }
    asm volatile("{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra WAIT_%=;\n}"
                 ::"r"(mb) : "memory");
    if (any_fused) __syncthreads();                       // fused rows (generic-proxy stores) visible
    // a quad of words per step: one conflict-free 16 B shared load per row group (the 36-word
    // row stride makes 4 B column loads 4-way bank conflicted), four 32x32 transposes
    uint32_t cms[LW];
#pragma unroll
    for (int g = 0; g < LW; ++g) cms[g] = s_cm[g * 32 + lane];
#pragma unroll
    for (uint32_t q = 0; q < PK_WPW / 4; ++q) {
        const uint32_t wq = wid * PK_WPW + q * 4;
        if (w0 + wq >= kb.W4) break;                       // W4 is a multiple of 8: whole quads
        if (!(ums[4 * q] | ums[4 * q + 1] | ums[4 * q + 2] | ums[4 * q + 3])) continue;   // warp-uniform
        uint32_t o[4][LW];
#pragma unroll
        for (int g = 0; g < LW; ++g) {
            if (rec == 1 && g >= 4) break;                 // a narrow pack: lanes 128.. are empty
            if ((uint32_t)g * 32 >= count) {               // lanes without a node: zero words, no transposes
                o[0][g] = o[1][g] = o[2][g] = o[3][g] = 0u;
                continue;
            }
            const uint4 v = *reinterpret_cast<const uint4 *>(sm + (g * 32 + lane) * PK_STRIDE + wq);
            o[0][g] = warp_transpose(v.x ^ cms[g], lane);
            o[1][g] = warp_transpose(v.y ^ cms[g], lane);
            o[2][g] = warp_transpose(v.z ^ cms[g], lane);
            o[3][g] = warp_transpose(v.w ^ cms[g], lane);
        }
#pragma unroll
        for (uint32_t kk = 0; kk < 4; ++kk) {
            const uint32_t w = w0 + wq + kk, um = ums[4 * q + kk];
            if (!umask) {
                const uint64_t y = (uint64_t)w * 32 + lane;
                HCHECK(rec * y + rec <= t_stride);
                T[rec * y] = make_uint4(o[kk][0], o[kk][1], o[kk][2], o[kk][3]);
                if (rec != 1) T[rec * y + 1] = make_uint4(o[kk][4], o[kk][5], o[kk][6], o[kk][7]);
            } else if ((um >> lane) & 1u) {
                const uint64_t t = ubs[4 * q + kk] + __popc(um & ((1u << lane) - 1u));
                HCHECK(2 * t + 2 <= t_stride);
                T[2 * t] = make_uint4(o[kk][0], o[kk][1], o[kk][2], o[kk][3]);
                T[2 * t + 1] = make_uint4(o[kk][4], o[kk][5], o[kk][6], o[kk][7]);
            }
        }
    }
}

// ------------------------------------------------------------------------------
// heavy rows: CTA (256 threads) per chunk of <= kHeavyChunk edges.  The threads form groups of
// G (1: a narrow pack of <= 128 nodes, 2: lane pairs for one pack, 4: quads for a pack pair),
// thread q of a group owns words 4q .. 4q+3 of the 4G-word lane record (pack q >> 1).
template <bool COUNT, int G>
__global__ void __launch_bounds__(256) k_slice_heavy(SliceDir dir, SliceScratch sc0, const RestrictDesc *__restrict__ d_run,
                                                     uint32_t run) {
    constexpr int NP = G < 2 ? 1 : G / 2, NG = 256 / G, RW = 4 * G;   // packs per pass, groups, record words
    const uint32_t p0 = blockIdx.y * NP;                  // first pack of this pass
    const SliceScratch sc = sc0.at(p0);
    const RestrictDesc *d = d_run + 256u * p0;
    const uint32_t count = min(256u * NP, run - 256u * p0);
    __shared__ PackConstN<NP> pc;
    __shared__ uint32_t red[8][G][COUNT ? NPL : 1][HW];
    __shared__ uint32_t fin[G][COUNT ? NPL : 1][HW];
    __shared__ uint32_t outw[NP * LW];
    __shared__ uint32_t s_last;
    const uint4 ch = dir.chunks[blockIdx.x];
    const uint32_t h = ch.x;
    HCHECK(h < dir.n_heavy && ch.y <= ch.z);
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, q = lane & (G - 1);
    Acc<COUNT> acc;
    acc.zero();
    scan_edges<COUNT, G>(acc, dir.col, sc.T, ch.y + threadIdx.x / G, ch.z, NG, q, sc.t_cap);
    acc.template warp_reduce_pairs<16, G>();
    if (lane < G)
        for (int c = 0; c < (COUNT ? NPL : 1); ++c)
            for (int k = 0; k < HW; ++k) red[wid][q][c][k] = acc.c[c][k];
    __syncthreads();
    if (threadIdx.x < G) {
        Acc<COUNT> a, b;
        for (int c = 0; c < (COUNT ? NPL : 1); ++c) for (int k = 0; k < HW; ++k) a.c[c][k] = red[0][threadIdx.x][c][k];
        for (int w = 1; w < 8; ++w) {
            for (int c = 0; c < (COUNT ? NPL : 1); ++c) for (int k = 0; k < HW; ++k) b.c[c][k] = red[w][threadIdx.x][c][k];
            a.merge(b);
        }
        for (int c = 0; c < (COUNT ? NPL : 1); ++c) for (int k = 0; k < HW; ++k) fin[threadIdx.x][c][k] = a.c[c][k];
    }
    __syncthreads();
    if (!COUNT) {
        if (threadIdx.x < RW) {                           // word kk of the pass: pack kk / 8, word kk % 8
            const uint32_t kk = threadIdx.x;
            const uint32_t x = fin[kk >> 2][0][kk & 3];
            if (x) atomicOr(sc0.at(p0 + (kk >> 3)).hacc + (size_t)h * LW + (kk & 7), x);
        }
    } else {
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
            const uint32_t L = threadIdx.x, LL = pp * 256 + L;   // lane of pack pp: half, word, bit
            if (LL >= 128u * G) continue;
            const uint32_t g = LL >> 7, k = (L >> 5) & 3, bit = L & 31;
            uint32_t val = 0;
            for (int c = 0; c < NPL; ++c) val |= ((fin[g][c][k] >> bit) & 1u) << c;
            if (val) atomicAdd(sc0.at(p0 + pp).hcnt + (size_t)h * 256 + L, val);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t t = atomicAdd(sc.ticket + h, 1u);
        s_last = (t == __ldg(dir.heavy_nchunks + h) - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    build_consts(pc, d, count);
    if (!COUNT) {
        if (threadIdx.x < RW) {
            const uint32_t kk = threadIdx.x;
            const SliceScratch sp = sc0.at(p0 + (kk >> 3));
            const uint32_t a = atomicExch(sp.hacc + (size_t)h * LW + (kk & 7), 0u);   // read + self-clean
            sp.hout[(size_t)h * LW + (kk & 7)] = ((a ^ pc.fl[kk]) & pc.am[kk]) | pc.om[kk];
        }
    } else {
        if (threadIdx.x < NP * LW) outw[threadIdx.x] = 0;
        __syncthreads();
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
            const uint32_t L = threadIdx.x;
            if (pp * 256 + L >= 128u * G) continue;
            uint32_t c = atomicExch(sc0.at(p0 + pp).hcnt + (size_t)h * 256 + L, 0u);
            c = c > 31u ? 31u : c;
            const uint32_t k = pp * LW + (L >> 5), bit = 1u << (L & 31);
            uint32_t n = 0;
            for (int cq = 0; cq < NPL; ++cq) n |= ((pc.nb[cq][k] & bit) ? 1u : 0u) << cq;
            bool r;
            if (pc.mge[k] & bit) r = c >= n;
            else if (pc.mle[k] & bit) r = c <= n;
            else if (pc.meq[k] & bit) r = c == n;
            else if (pc.mlep[k] & bit) r = c > 0 && c <= n;
            else r = false;
            if (r) atomicOr(&outw[k], bit);
        }
        __syncthreads();
        if (threadIdx.x < RW) sc0.at(p0 + (threadIdx.x >> 3)).hout[(size_t)h * LW + (threadIdx.x & 7)] = outw[threadIdx.x];
    }
    if (threadIdx.x == 0) sc.ticket[h] = 0;
}

// ------------------------------------------------------------------------------
// acc += T[y] over the neighbours of one row split across S lane pairs (this pair takes
// edges e, e+S, e+2S, ... below b).  Software-pipelined: the next step's four neighbour
// indices are loaded before this step's four T gathers, so the CSR stream (DRAM) and the
// T gathers (L2) overlap instead of adding up.
template <bool COUNT, int R = 2>
__device__ __forceinline__ void scan_strided(Acc<COUNT> &acc, const uint32_t *__restrict__ col, const uint4 *__restrict__ T,
                                             uint32_t e, uint32_t b, uint32_t S, uint32_t half, uint64_t cap) {
    uint32_t y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) y[u] = e + S * u < b ? __ldg(col + e + S * u) : 0xffffffffu;
    for (; e < b; e += 4 * S) {
        uint32_t yn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) yn[u] = e + S * (4 + u) < b ? __ldg(col + e + S * (4 + u)) : 0xffffffffu;
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            HCHECK(y[u] == 0xffffffffu || (uint64_t)R * y[u] + R <= cap);
            v[u] = y[u] != 0xffffffffu ? __ldg(T + (uint64_t)R * y[u] + half) : make_uint4(0, 0, 0, 0);
        }
        acc.add4(v[0], v[1], v[2], v[3]);
#pragma unroll
        for (int u = 0; u < 4; ++u) y[u] = yn[u];
    }
}

// one SELL-16 slice (16 rows of similar degree, neighbour k of row i at c[16k + i]), a lane
// pair per row, the same software pipeline over the slice's width w (a multiple of 4)
template <bool COUNT, int R = 2>
__device__ __forceinline__ void scan_slice_pipelined(Acc<COUNT> &acc, const uint32_t *__restrict__ c, const uint4 *__restrict__ T,
                                                     uint32_t w, uint32_t half, uint64_t cap) {
    if (!w) return;
    uint32_t y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) y[u] = __ldg(c + u * 16);
    for (uint32_t k = 0; k < w; k += 4) {
        uint32_t yn[4];
        const bool more = k + 4 < w;
#pragma unroll
        for (int u = 0; u < 4; ++u) yn[u] = more ? __ldg(c + (k + 4 + u) * 16) : 0xffffffffu;
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            HCHECK(y[u] == 0xffffffffu || (uint64_t)R * y[u] + R <= cap);
            v[u] = y[u] != 0xffffffffu ? __ldg(T + (uint64_t)R * y[u] + half) : make_uint4(0, 0, 0, 0);
        }
        acc.add4(v[0], v[1], v[2], v[3]);
#pragma unroll
        for (int u = 0; u < 4; ++u) y[u] = yn[u];
    }
}

// ------------------------------------------------------------------------------
// Persistent sweep over 1024-individual tiles (grid = resident CTAs).  G threads per row
// ("Narrow packs"): thread q of a row's group owns words 4q .. 4q+3 of
// the row's 4G-word lane record (T record of 16 G bytes, one gather per edge and group):
// G = 1 a narrow pack (<= 128 nodes), 2 one pack, 4 a pack pair (512-thread CTAs).  CTAs take tiles from a global counter in
// decreasing-cost order (dir.tile_rank, LPT), and inside a tile the warps take work items
// (medium rows, then SELL slices, both degree-descending) from a shared counter, so neither
// the grid nor the CTA waits on a statically unlucky share.  The counter pair `sched` is
// self-cleaning: the last CTA to finish resets it for the next launch on the stream.
template <bool COUNT, int G>
__global__ void __launch_bounds__(G == 4 ? 512 : 256, G == 4 ? 2 : 4) k_slice_tile(KbDev kb, SliceDir dir, SliceScratch sc, UTab ut,
                                                                 const RestrictDesc *__restrict__ d, uint32_t count,
                                                                 hedl_counts *counts, uint32_t *sched, uint32_t dbg) {
#ifndef HEDL_DEBUG_TILE
    dbg = 0;                                              // release builds: the debug switches fold away
#endif
    constexpr int NP = G < 2 ? 1 : G / 2;                 // packs of the pass
    constexpr uint32_t RW = 4 * G;                        // record words (lanes / 32)
    constexpr uint32_t TR = RW + 1;                       // ot row stride (bank-conflict-free transposes)
    constexpr uint32_t NT = G == 4 ? 512 : 256;
    extern __shared__ uint32_t smem[];
    PackConstN<NP> &pc = *reinterpret_cast<PackConstN<NP> *>(smem);
    uint32_t *ot = smem + sizeof(PackConstN<NP>) / 4;     // [1024][TR]
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, q = lane & (G - 1);
    __shared__ uint32_t s_exm[32], s_exb[32];
    __shared__ uint32_t s_tile, s_item;
    __shared__ uint32_t s_udirs;
    // this lane's node for the transpose-back phase (fixed for the whole launch): warp g takes
    // record word (column) g; a narrow pack's 4 columns go to warps w and w + 4 (word halves)
    const uint32_t jn = (G == 1 ? (wid & 3) : wid) * 32 + lane;
    uint32_t *r_out = nullptr, *r_proj = nullptr, *r_uout = nullptr;
    uint32_t r_udirs = 0;
    int32_t r_cover = -1;
    if (jn < count) {
        r_out = d[jn].out;
        r_proj = d[jn].proj;
        r_cover = d[jn].cover;
        r_uout = d[jn].uout;
        r_udirs = r_uout ? d[jn].udirs : 0u;
    }
    if (threadIdx.x == 0) s_udirs = 0;
    __syncthreads();
    if (r_udirs) atomicOr(&s_udirs, r_udirs);            // directions some node of the pass emits
    build_consts(pc, d, count);                           // (contains __syncthreads)
    const bool live = jn < count;
    uint32_t tp = 0, fp = 0;
    for (;;) {
        __syncthreads();                                  // previous tile's transpose-back done
        if (threadIdx.x == 0) {
            s_tile = atomicAdd(sched, 1u);
            s_item = 0;
        }
        __syncthreads();
        const uint32_t tt = s_tile;
        if (tt >= dir.n_tiles) break;
        const uint32_t t = __ldg(dir.tile_rank + tt);
        const uint32_t x0 = t * 1024;
        if (x0 + 1024 > kb.N)                              // only the last tile has rows >= N (left 0)
            for (uint32_t i = threadIdx.x; i < 1024 * TR; i += NT) ot[i] = 0;
        if (threadIdx.x < 32) {
            const uint32_t w = t * 32 + threadIdx.x;
            s_exm[threadIdx.x] = w < kb.W ? __ldg(kb.ex_mask + w) : 0u;
            s_exb[threadIdx.x] = w < kb.W ? __ldg(kb.ex_base + w) : 0u;
        }
        const uint4 ti = dir.tiles[t];
        const uint32_t hbeg = ti.w, hend = dir.tiles[t + 1].w;
        if (x0 + 1024 > kb.N) __syncthreads();            // zero fill before the heavy rows land
        for (uint32_t h = hbeg + threadIdx.x; h < hend; h += NT) {
            const uint32_t xl = __ldg(dir.heavy_x + h) - x0;
            HCHECK(xl < 1024u);
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) {
                const uint32_t *ho = sc.at(pp).hout + (size_t)h * LW;
#pragma unroll
                for (int k = 0; k < (RW < LW ? (int)RW : LW); ++k) ot[xl * TR + pp * LW + k] = ho[k];
            }
        }
        const uint32_t sbeg = __ldg(dir.tile_slice + t), send = __ldg(dir.tile_slice + t + 1);
        // work items, in this order: big medium rows (deg > kMidDeg; a warp each), mid rows
        // (4 per warp, 8 lanes each), light SELL-16 slices (SPI per item; for a pack pair a
        // slice's 16 rows are two 8-row halves of the warp)
        constexpr uint32_t SPI = G == 1 ? 2u : (COUNT || G == 4) ? 1u : 2u;
        const uint32_t n_big = (dbg & 2) ? 0u : __ldg(dir.tile_nbig + t);
        const uint32_t n_med = (dbg & 2) ? 0u : ti.y, n_sl = (dbg & 1) ? 0u : send - sbeg;
        const uint32_t i_light = n_big + (n_med - n_big + 3) / 4;
        const uint32_t n_items = i_light + (n_sl + SPI - 1) / SPI;
        uint32_t nxt = 0;
        if (lane == 0) nxt = atomicAdd(&s_item, 1u);
        nxt = __shfl_sync(FULL, nxt, 0);
        while (nxt < n_items) {
            const uint32_t it = nxt;
            if (lane == 0) nxt = atomicAdd(&s_item, 1u);  // the next item, fetched under this one
            Acc<COUNT> acc;
            acc.zero();
            if (it < n_big) {
                // big medium row: warp per row, the 32 / G thread groups split its neighbours
                const uint32_t x = __ldg(dir.order + ti.x + it);
                HCHECK(x - x0 < 1024u);
                const uint32_t a = __ldg(dir.row_ptr + x), b = __ldg(dir.row_ptr + x + 1);
                scan_strided<COUNT, G>(acc, dir.col, sc.T, a + lane / G, b, 32 / G, q, sc.t_cap);
                acc.template warp_reduce_pairs<16, G>();
                if (lane < G) {
#pragma unroll
                    for (int k = 0; k < HW; ++k) ot[(x - x0) * TR + q * HW + k] = acc.result(pc, q * HW + k, k);
                }
            } else if (it < i_light) {
                // mid rows: 4 per warp, the 8 / G groups of each 8-lane block split one row
                const uint32_t p = (lane / G) & (8 / G - 1);
                const uint32_t mi = n_big + (it - n_big) * 4 + (lane >> 3);
                const bool rv = mi < n_med;
                uint32_t x = 0, a = 0, b = 0;
                if (rv) {
                    x = __ldg(dir.order + ti.x + mi);
                    HCHECK(x - x0 < 1024u);
                    a = __ldg(dir.row_ptr + x);
                    b = __ldg(dir.row_ptr + x + 1);
                }
                scan_strided<COUNT, G>(acc, dir.col, sc.T, a + p, b, 8 / G, q, sc.t_cap);
                acc.template warp_reduce_pairs<4, G>();
                if (rv && p == 0) {
#pragma unroll
                    for (int k = 0; k < HW; ++k) ot[(x - x0) * TR + q * HW + k] = acc.result(pc, q * HW + k, k);
                }
            } else if (G == 1) {
                // light rows of a narrow pack: a thread per row, the warp's halves on two SELL-16
                // slices (16 consecutive neighbour indices per half and step, coalesced)
                const uint32_t sl = (it - i_light) * 2 + (lane >> 4);
                const bool sv = sl < n_sl;
                const uint32_t li = sl * 16 + (lane & 15);
                const bool rv = sv && li < ti.z;
                const uint32_t x = rv ? __ldg(dir.order + ti.x + ti.y + li) : 0u;
                HCHECK(!rv || x - x0 < 1024u);
                const uint32_t *c = sv ? dir.sell_col + __ldg(dir.sell_off + sbeg + sl) + (lane & 15) : dir.sell_col;
                scan_slice_pipelined<COUNT, G>(acc, c, sc.T, sv ? __ldg(dir.sell_w + sbeg + sl) : 0u, 0u, sc.t_cap);
                if (rv) {
#pragma unroll
                    for (int k = 0; k < HW; ++k) ot[(x - x0) * TR + k] = acc.result(pc, k, k);
                }
            } else if (G == 2 && SPI == 1) {
                // light rows: one SELL-16 slice, a lane pair per row; the 16 pairs read 16
                // consecutive neighbour indices per step (coalesced)
                const uint32_t sl = it - i_light;
                const uint32_t li = sl * 16 + (lane >> 1);
                const bool rv = li < ti.z;
                const uint32_t x = rv ? __ldg(dir.order + ti.x + ti.y + li) : 0u;
                HCHECK(!rv || x - x0 < 1024u);
                const uint32_t *c = dir.sell_col + __ldg(dir.sell_off + sbeg + sl) + (lane >> 1);
                scan_slice_pipelined<COUNT, G>(acc, c, sc.T, __ldg(dir.sell_w + sbeg + sl), q, sc.t_cap);
                if (rv) {
#pragma unroll
                    for (int k = 0; k < HW; ++k) ot[(x - x0) * TR + q * HW + k] = acc.result(pc, q * HW + k, k);
                }
            } else if (G == 4 && COUNT) {
                // light rows of a pack pair, COUNT class: one SELL-16 slice, a quad per row, the
                // two 8-row halves one after the other (register budget)
                const uint32_t sl = it - i_light;
                const uint32_t *cb = dir.sell_col + __ldg(dir.sell_off + sbeg + sl) + (lane >> 2);
                const uint32_t wdt = __ldg(dir.sell_w + sbeg + sl);
#pragma unroll 1
                for (uint32_t hh = 0; hh < 2; ++hh) {
                    const uint32_t li = sl * 16 + hh * 8 + (lane >> 2);
                    const bool rv = li < ti.z;
                    const uint32_t x = rv ? __ldg(dir.order + ti.x + ti.y + li) : 0u;
                    HCHECK(!rv || x - x0 < 1024u);
                    if (hh) acc.zero();
                    scan_slice_pipelined<COUNT, G>(acc, cb + hh * 8, sc.T, wdt, q, sc.t_cap);
                    if (rv) {
#pragma unroll
                        for (int k = 0; k < HW; ++k) ot[(x - x0) * TR + q * HW + k] = acc.result(pc, q * HW + k, k);
                    }
                }
            } else {
                // light rows, OR class: two row sets per step, their dependent load chains (slice
                // bounds, neighbour ids, T gathers) overlapping -- one pack: two SELL-16 slices,
                // a lane pair per row; a pack pair: the two 8-row halves of one slice, a quad
                // per row
                Acc<COUNT> acc2;
                acc2.zero();
                uint32_t x[2], w[2];
                const uint32_t *cp[2];
                bool rv[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t sl = G == 2 ? (it - i_light) * 2 + h : it - i_light;
                    const bool sv = sl < n_sl;
                    const uint32_t li = G == 2 ? sl * 16 + (lane >> 1) : sl * 16 + h * 8 + (lane >> 2);
                    rv[h] = sv && li < ti.z;
                    x[h] = rv[h] ? __ldg(dir.order + ti.x + ti.y + li) : 0u;
                    HCHECK(!rv[h] || x[h] - x0 < 1024u);
                    const uint32_t col0 = G == 2 ? (lane >> 1) : h * 8 + (lane >> 2);
                    cp[h] = sv ? dir.sell_col + __ldg(dir.sell_off + sbeg + sl) + col0 : dir.sell_col;
                    w[h] = sv ? __ldg(dir.sell_w + sbeg + sl) : 0u;
                }
                const uint32_t wm = max(w[0], w[1]);
                for (uint32_t k = 0; k < wm; k += 4) {
                    uint32_t y[2][4];
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int u = 0; u < 4; ++u) y[h][u] = k < w[h] ? __ldg(cp[h] + (k + u) * 16) : 0xffffffffu;
                    uint4 v[2][4];
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            HCHECK(y[h][u] == 0xffffffffu || (uint64_t)G * y[h][u] + G <= sc.t_cap);
                            v[h][u] = y[h][u] != 0xffffffffu ? __ldg(sc.T + (uint64_t)G * y[h][u] + q) : make_uint4(0, 0, 0, 0);
                        }
                    acc.add4(v[0][0], v[0][1], v[0][2], v[0][3]);
                    acc2.add4(v[1][0], v[1][1], v[1][2], v[1][3]);
                }
                if (rv[0]) {
#pragma unroll
                    for (int k = 0; k < HW; ++k) ot[(x[0] - x0) * TR + q * HW + k] = acc.result(pc, q * HW + k, k);
                }
                if (rv[1]) {
#pragma unroll
                    for (int k = 0; k < HW; ++k) ot[(x[1] - x0) * TR + q * HW + k] = acc2.result(pc, q * HW + k, k);
                }
            }
            nxt = __shfl_sync(FULL, nxt, 0);
        }
        __syncthreads();
        // transpose back: warp g writes lanes 32g..32g+31 (node rows); each lane writes one
        // whole 32 B sector of its node's row per 8 words (a narrow pack: warps g and g + 4 take
        // the two 16-word halves of the tile)
        const uint32_t g = G == 1 ? (wid & 3) : wid;
        const uint32_t wl0 = G == 1 ? (wid >> 2) * 16 : 0u, wl1 = G == 1 ? wl0 + 16 : 32u;
        uint32_t pw = 0, pbits = 0;                       // pending projected word of this lane's node
        for (uint32_t wl = wl0; wl < ((dbg & 4) ? 0u : wl1); wl += 8) {
            const uint32_t w = t * 32 + wl;
            if (w >= kb.W4) break;                         // W4 is a multiple of 8
            uint32_t o[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = warp_transpose(ot[((wl + k) * 32 + lane) * TR + g], lane);
            if (live) {
                if (r_out) {
                    uint4 *dst = reinterpret_cast<uint4 *>(r_out + w);
                    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
                    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
                }
                if (r_proj) {
                    // example bits of word w+k -> the projected row (pext with the staged masks)
#pragma unroll
                    for (int k = 0; k < 8; ++k) pack_bits(s_exm[wl + k], o[k], s_exb[wl + k], r_proj, pw, pbits);
                }
                if (r_cover >= 0) {
                    const uint4 *pp = reinterpret_cast<const uint4 *>(kb.pos + w);
                    const uint4 *nn = reinterpret_cast<const uint4 *>(kb.neg + w);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const uint4 pv = __ldg(pp + hh), nv = __ldg(nn + hh);
                        const uint32_t *oo = o + 4 * hh;
                        tp += __popc(oo[0] & pv.x) + __popc(oo[1] & pv.y) + __popc(oo[2] & pv.z) + __popc(oo[3] & pv.w);
                        fp += __popc(oo[0] & nv.x) + __popc(oo[1] & nv.y) + __popc(oo[2] & nv.z) + __popc(oo[3] & nv.w);
                    }
                }
            }
        }
        if (pbits) atomicOr(r_proj + pw, pbits);
        // U rows: for each direction d some node of the pass
        // emits, the tile's members of U_d (the example rows' neighbours in direction d) are the
        // consecutive U positions [bl, bh) whose individuals ulist_d gives; 32 of them at a time,
        // their result rows (ot) go through one more warp transpose, and lane j of warp g holds
        // node 32g + j's U word.  Interior U words are written whole, the two seam words shared
        // with the neighbouring tiles by atomicOr into the zeroed row.  (No block barrier: ot is
        // stable until the next tile's first __syncthreads.  Selecting the members from the
        // tile's U-mask words with warp scans instead of the ulist loads measured 2% slower.)
#pragma unroll
        for (uint32_t dd = 0; dd < kMaxUDirs; ++dd) {
            if (!((s_udirs >> dd) & 1u)) continue;                        // block-uniform
            if (G == 1 && wid >= 4) break;                                // a narrow pack: 4 columns
            const uint32_t bl = __ldg(ut.ub[dd] + t * 32);
            const uint32_t bh = t * 32 + 32 < kb.W4 ? __ldg(ut.ub[dd] + t * 32 + 32) : ut.nu[dd];
            if (bh <= bl) continue;
            const bool mine = live && ((r_udirs >> dd) & 1u);
            uint32_t *urow = mine ? r_uout + __popc(r_udirs & ((1u << dd) - 1u)) * ut.stride : nullptr;
            const uint32_t c0 = bl >> 5, c1 = (bh - 1) >> 5;
            for (uint32_t cw = c0; cw <= c1; ++cw) {
                const uint32_t pos = cw * 32 + lane;
                HCHECK(!(pos >= bl && pos < bh) || (pos < ut.nu[dd] && __ldg(ut.ul[dd] + pos) - x0 < 1024u));
                const uint32_t v = (pos >= bl && pos < bh) ? ot[(__ldg(ut.ul[dd] + pos) - x0) * TR + g] : 0u;
                const uint32_t x = warp_transpose(v, lane);
                if (mine) {
                    const bool seam = (cw == c0 && (bl & 31)) || (cw == c1 && (bh & 31));
                    if (seam) { if (x) atomicOr(urow + cw, x); }
                    else urow[cw] = x;
                }
            }
        }
    }
    // coverage of this CTA's tiles, one atomic set per node per CTA
    if (live && r_cover >= 0 && (tp | fp)) {
        hedl_counts *c = counts + r_cover;
        if (tp) {
            atomicAdd((unsigned long long *)&c->tp, (unsigned long long)tp);
            atomicAdd((unsigned long long *)&c->fn, 0ull - tp);
        }
        if (fp) {
            atomicAdd((unsigned long long *)&c->fp, (unsigned long long)fp);
            atomicAdd((unsigned long long *)&c->tn, 0ull - fp);
        }
    }
    // self-cleaning scheduler: the last CTA out resets the counters for the next launch
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
            sched[0] = 0;
            sched[1] = 0;
            __threadfence();
        }
    }
}

// ------------------------------------------------------------------------------
// EX packs: only the example rows (ranks of E); 128 ranks per CTA; the result goes
// straight to the nodes' example-projected rows (4 projected words per CTA, owned:
// plain stores) with fused coverage against the projected example masks.
struct ExArgs {
    const uint32_t *erp, *ecol;       // example-row CSR over ranks, neighbours as compact T indices
    const uint4 *ex_tiles;
    const uint32_t *ex_order, *ex_ids, *ex_hrank;
    const uint32_t *ppos, *pneg;
    uint32_t MW4;
};

template <bool COUNT>
__global__ void __launch_bounds__(256, COUNT ? 4 : 6) k_slice_ex(ExArgs a, SliceScratch sc0, const RestrictDesc *__restrict__ d_run,
                                                                 uint32_t run, hedl_counts *counts) {
    const SliceScratch sc = sc0.at(blockIdx.y);
    const RestrictDesc *d = d_run + 256u * blockIdx.y;
    const uint32_t count = pack_count(run, blockIdx.y);
    __shared__ PackConst pc;
    __shared__ uint32_t ot[128 * TROW];
    const uint32_t b = blockIdx.x, r0 = b * 128;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, half = lane & 1;
    for (uint32_t i = threadIdx.x; i < 128 * TROW; i += 256) ot[i] = 0;
    build_consts(pc, d, count);                           // (contains __syncthreads)
    const uint4 ti = a.ex_tiles[b];
    const uint32_t hbeg = ti.w, hend = a.ex_tiles[b + 1].w;
    for (uint32_t h = hbeg + threadIdx.x; h < hend; h += 256) {
        const uint32_t rl = __ldg(a.ex_hrank + h) - r0;
        HCHECK(rl < 128u);
#pragma unroll
        for (int k = 0; k < LW; ++k) ot[rl * TROW + k] = sc.hout[(size_t)h * LW + k];
    }
    for (uint32_t m = wid; m < ti.y; m += 8) {            // medium rows: warp per row
        const uint32_t r = __ldg(a.ex_order + ti.x + m);
        HCHECK(r - r0 < 128u);
        const uint32_t e0 = __ldg(a.erp + r), e1 = __ldg(a.erp + r + 1);
        Acc<COUNT> acc;
        acc.zero();
        scan_edges<COUNT>(acc, a.ecol, sc.T, e0 + (lane >> 1), e1, 16, half, sc.t_cap);
        acc.template warp_reduce_pairs<16>();
        if (lane < 2) {
#pragma unroll
            for (int k = 0; k < HW; ++k) ot[(r - r0) * TROW + half * HW + k] = acc.result(pc, half * HW + k, k);
        }
    }
    for (uint32_t l = threadIdx.x >> 1; l < ti.z; l += 128) {   // light rows: lane pair per row
        const uint32_t r = __ldg(a.ex_order + ti.x + ti.y + l);
        HCHECK(r - r0 < 128u);
        const uint32_t e0 = __ldg(a.erp + r), e1 = __ldg(a.erp + r + 1);
        Acc<COUNT> acc;
        acc.zero();
        scan_edges<COUNT>(acc, a.ecol, sc.T, e0, e1, 1, half, sc.t_cap);
#pragma unroll
        for (int k = 0; k < HW; ++k) ot[(r - r0) * TROW + half * HW + k] = acc.result(pc, half * HW + k, k);
    }
    __syncthreads();
    const uint32_t g = wid, j = g * 32 + lane;
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = warp_transpose(ot[(q * 32 + lane) * TROW + g], lane);
    if (j >= count) return;                               // (after the warp-wide transposes)
    const RestrictDesc r = d[j];
    const uint32_t w = b * 4;
    if (r.proj) *reinterpret_cast<uint4 *>(r.proj + w) = make_uint4(o[0], o[1], o[2], o[3]);
    if (r.cover >= 0) {
        const uint4 p = __ldg(reinterpret_cast<const uint4 *>(a.ppos + w));
        const uint4 n = __ldg(reinterpret_cast<const uint4 *>(a.pneg + w));
        const uint32_t tp = __popc(o[0] & p.x) + __popc(o[1] & p.y) + __popc(o[2] & p.z) + __popc(o[3] & p.w);
        const uint32_t fp = __popc(o[0] & n.x) + __popc(o[1] & n.y) + __popc(o[2] & n.z) + __popc(o[3] & n.w);
        hedl_counts *c = counts + r.cover;
        if (tp) {
            atomicAdd((unsigned long long *)&c->tp, (unsigned long long)tp);
            atomicAdd((unsigned long long *)&c->fn, 0ull - tp);
        }
        if (fp) {
            atomicAdd((unsigned long long *)&c->fp, (unsigned long long)fp);
            atomicAdd((unsigned long long *)&c->tn, 0ull - fp);
        }
    }
}

inline uint32_t cdiv(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }
}  // namespace

bool slice_enabled(const hedl_kb *kb) { return kb->N > 0; }

bool slice_worthwhile(const hedl_kb *, uint32_t n_nodes, bool force) { return n_nodes >= (force ? 1u : kSliceMinNodes); }

uint32_t slice_class(uint32_t pred, uint32_t n, uint32_t sat) {
    if (sat <= 1) return 0;                  // OR pack
    if (n <= 30 && sat <= 31) return 1;      // COUNT pack
    (void)pred;
    return 2;                                // per-node kernel
}

namespace {
// One fixed scratch layout for every direction of the KB (sized by the largest heavy lists),
// so the self-cleaning accumulators of one direction never alias another's results:
//   [T x max_batch][full-pack heavy scratch (nh)][EX heavy scratch (max_batch x nhx)][sched]
struct SliceLayout {
    size_t t_bytes, tx_bytes, off_hf, off_hx, need, nh, nhx;
    uint32_t max_batch;
};
SliceLayout slice_layout(const hedl_kb *kb) {
    SliceLayout L;
    L.t_bytes = (size_t)kb->W4 * 32 * 32;                 // full packs: 32 B per individual
    size_t nu_max = 0;
    for (const hedl_dir &x : kb->dirs) nu_max = std::max<size_t>({nu_max, (size_t)x.n_u, (size_t)x.UW4 * 32});
    L.tx_bytes = std::max<size_t>(nu_max * 32, 256);      // EX packs: 32 B per neighbour of an example
    L.nh = L.nhx = 0;
    for (const hedl_dir &x : kb->dirs) {
        L.nh = std::max<size_t>(L.nh, x.n_heavy);
        L.nhx = std::max<size_t>(L.nhx, x.n_ex_heavy);
        for (const hedl_rowset &rs : x.usw) L.nhx = std::max<size_t>(L.nhx, rs.n_heavy);
    }
    const size_t per_h = (LW + 256 + 1 + LW) * 4;
    L.max_batch = (uint32_t)std::max<size_t>(1, std::min<size_t>(128, (4ull << 30) / L.tx_bytes));
    // full packs go in pairs: room for two packs' T and heavy scratch
    L.off_hf = std::max(2 * L.t_bytes, L.tx_bytes * L.max_batch);
    L.off_hx = L.off_hf + 2 * L.nh * per_h;
    L.need = L.off_hx + (size_t)L.max_batch * L.nhx * per_h + 256;
    return L;
}
}  // namespace

size_t slice_ws_bytes(const hedl_kb *kb) { return slice_layout(kb).need; }

hedl_status slice_run(const hedl_kb *kb, void **ws, size_t *ws_bytes, cudaStream_t s, const KbDev &kd, uint32_t dirid,
                      const RestrictDesc *h_desc, const RestrictDesc *d_desc, uint32_t n, hedl_counts *counts, bool ex,
                      int fixed_cls, bool ucomp, const Operand *d_ops, int usw) {
    const hedl_dir &dr = kb->dirs[dirid];
    if (ex && !kb->M) return HEDL_OK;                     // no examples: nothing to evaluate
    const SliceLayout lay = slice_layout(kb);
    const size_t t_bytes = lay.t_bytes, tx_bytes = lay.tx_bytes;
    const size_t nh = lay.nh, nhx = lay.nhx, off_hf = lay.off_hf, off_hx = lay.off_hx, need = lay.need;
    const uint32_t max_batch = lay.max_batch;
    if (*ws_bytes < need) {
        // a buffer being replaced may still be read by launched kernels; a fresh one (the first
        // evaluation of a program) needs no synchronisation -- the launches keep streaming
        if (*ws) {
            HEDL_CUDA(kb, cudaStreamSynchronize(s));
            dev_free(*ws, s);
        }
        *ws = nullptr;
        *ws_bytes = 0;
        size_t got = 0;
        if (void *q = pool_take(kb, PR_SLICE, need, &got)) {   // self-cleaned accumulators
            *ws = q;
            *ws_bytes = got;
        } else {
            if (dev_malloc(ws, need, s) != cudaSuccess) { cudaGetLastError(); *ws = nullptr; return fail(HEDL_ERR_OOM, "slice workspace"); }
            HEDL_CUDA(kb, cudaMemsetAsync(*ws, 0, need, s));
            *ws_bytes = need;
        }
    }
    char *base = (char *)*ws;
    // field-major accumulators with room for `npacks` packs of `nrows` heavy rows each
    auto scratch = [&](size_t off, size_t nrows, size_t npacks) {
        const size_t cap = nrows * npacks;
        SliceScratch sc;
        sc.T = (uint4 *)base;
        sc.hacc = (uint32_t *)(base + off);
        sc.hcnt = sc.hacc + cap * LW;
        sc.ticket = sc.hcnt + cap * 256;
        sc.hout = sc.ticket + cap;
        sc.t_stride = t_bytes / 16;
        sc.t_cap = t_bytes / 16;
        sc.h_stride = 0;
        return sc;
    };
    SliceDir sd{dr.row_ptr, dr.col, dr.tiles, dr.order, dr.tile_rank, dr.tile_nbig, dr.tile_slice, dr.sell_off, dr.sell_w, dr.sell_col,
                dr.heavy_x, dr.heavy_nchunks, dr.chunks, dr.n_heavy, dr.n_chunks, dr.n_tiles};
    SliceDir sdx{dr.ex_rp, dr.ex_ccol, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                 dr.ex_hx, dr.ex_hn, dr.ex_chunks, dr.n_ex_heavy, dr.n_ex_chunks, 0};
    const ExArgs xa{dr.ex_rp, dr.ex_ccol, dr.ex_tiles, dr.ex_order, kb->ex_ids, dr.ex_hrank, kb->ppos, kb->pneg, kb->MW4};
    const size_t smem = sizeof(PackConst) + 1024 * TROW * 4;
    const size_t smem2 = sizeof(PackConstN<2>) + 1024 * (2 * LW + 1) * 4;   // pack pairs (2 CTAs/SM)
    const size_t smem1 = sizeof(PackConst) + 1024 * (LW / 2 + 1) * 4;        // narrow packs
    const size_t pk_smem = 256 * PK_STRIDE * 4;
    static std::once_flag attr_set[kMaxDevices];
    once_per_device(attr_set, [&] {
        // shared-memory carveout: just enough for 4 resident CTAs, the rest of the 256 KB
        // L1/shared array stays L1 (the T gathers run at half rate with the minimum L1:
        // tools/gather_bench.cu)
        int dev = 0, maxsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        auto carve = [&](const void *f, size_t dyn, int ctas) {
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, f);
            const double need = (double)ctas * (double)(dyn + fa.sharedSizeBytes + 1024);
            int pct = maxsm > 0 ? (int)std::ceil(100.0 * need / maxsm) : 100;
            pct = std::max(0, std::min(100, pct));
            cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
        };
        cudaFuncSetAttribute(k_slice_tile<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_slice_tile<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        carve((const void *)k_slice_tile<false, 2>, smem, 4);
        carve((const void *)k_slice_tile<true, 2>, smem, 4);
        cudaFuncSetAttribute(k_slice_tile<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        cudaFuncSetAttribute(k_slice_tile<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        carve((const void *)k_slice_tile<false, 4>, smem2, 2);
        carve((const void *)k_slice_tile<true, 4>, smem2, 2);
        carve((const void *)k_slice_tile<false, 1>, smem1, 4);
        carve((const void *)k_slice_tile<true, 1>, smem1, 4);
        cudaFuncSetAttribute(k_slice_pack, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pk_smem);
        carve((const void *)k_slice_pack, pk_smem, 4);
    });
    const double csr = 4.0 * (kb->N + 1) + 4.0 * dr.E;
    for (uint32_t off = 0; off < n;) {
        // a run of consecutive same-class descriptors: full packs go one pack per launch
        // (T stays L2-resident for the tile sweep); EX packs go up to max_batch per launch
        const uint32_t cls = fixed_cls >= 0 ? (uint32_t)fixed_cls : slice_class(h_desc[off].pred, h_desc[off].n, h_desc[off].sat);
        // U sweeps: full T per pack, as many packs per launch as the T area holds
        const uint32_t usw_batch = (uint32_t)std::max<size_t>(1, std::min<size_t>(max_batch, off_hf / std::max<size_t>(t_bytes, 1)));
        // full packs: two per CSR pass (pack pairs) unless HEDL_NO_PAIR (A/B)
        static const bool no_pair = std::getenv("HEDL_NO_PAIR") != nullptr;
        const uint32_t cap = ex ? 256u * max_batch : usw >= 0 ? 256u * usw_batch : (no_pair ? 256u : 512u);
        uint32_t run = 1;
        if (fixed_cls >= 0) run = std::min(n - off, cap);
        else
            while (off + run < n && run < cap &&
                   slice_class(h_desc[off + run].pred, h_desc[off + run].n, h_desc[off + run].sat) == cls)
                ++run;
        const uint32_t packs = (run + 255) / 256;
        const RestrictDesc *dd = d_desc + off;
        SliceScratch sc = (ex || usw >= 0) ? scratch(off_hx, nhx, max_batch) : scratch(off_hf, nh, 2);
        const bool pair = !ex && usw < 0 && packs == 2;
        // narrow packs: a full pack of <= 128 nodes sweeps with one
        // thread per row and 16 B T records; HEDL_NO_NARROW=1 disables (A/B)
        static const bool no_narrow = std::getenv("HEDL_NO_NARROW") != nullptr;
        const bool narrow = !ex && usw < 0 && packs == 1 && run <= 128 && !no_narrow;
        if (pair) {
            sc.h_stride = nh;                             // the two packs' heavy accumulators
            sc.t_stride = 2 * t_bytes / 16;               // one interleaved region of 64 B records
            sc.t_cap = 2 * t_bytes / 16;
        } else if (narrow) {
            sc.t_stride = t_bytes / 32;                   // 16 B records
            sc.t_cap = t_bytes / 32;
        }
        if (ex) {
            sc.h_stride = nhx;
            sc.t_stride = tx_bytes / 16;
            sc.t_cap = tx_bytes / 16;
        } else if (usw >= 0) {
            sc.h_stride = nhx;                            // (t_stride: one full T per pack)
        }
        prof_begin(s, KC_SLICE_IN);
        if (ex && ucomp) {
            // fillers are U rows: pack them whole (T index = U index), no compaction
            KbDev ku = kd;
            ku.W4 = dr.UW4;
            if (dr.UW4)
                k_slice_pack<<<dim3(cdiv(dr.UW4, PK_WORDS), packs), 256, pk_smem, s>>>(ku, dd, run, sc.T, sc.t_stride,
                                                                                     nullptr, nullptr, nullptr, 2u);
            count_launch();
            prof_end(s, KC_SLICE_IN, 4.0 * dr.UW * run + 32.0 * dr.n_u * packs, packs);
        } else {
            k_slice_pack<<<dim3(cdiv(kb->W4, PK_WORDS), packs), 256, pk_smem, s>>>(kd, dd, run, sc.T, sc.t_stride,
                                                                                 ex ? dr.ex_umask : nullptr,
                                                                                 ex ? dr.ex_ubase : nullptr, d_ops,
                                                                                 pair ? 4u : narrow ? 1u : 2u);
            count_launch();
            // rows read: one per materialised filler, the operand rows of a fused one
            double rows_read = run;
            if (h_desc)
                for (uint32_t j = 0; j < run; ++j)
                    if (!h_desc[off + j].child) rows_read += (double)(h_desc[off + j].op_n & 0x7fffffffu) - 1.0;
            prof_end(s, KC_SLICE_IN, 4.0 * kb->W * rows_read + 32.0 * (ex ? (double)dr.n_u : 32.0 * kb->W4) * packs, packs);
        }
        if (usw >= 0) {
            // U sweep: the pack's nodes are needed only over U_usw, so only
            // the rows of U_usw are swept -- the example-row sweep over that row set, writing the
            // nodes' U rows (RestrictDesc.proj) instead of projected rows
            const hedl_rowset &rs = dr.usw[usw];
            const SliceDir su{rs.rp, rs.col, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                              rs.hx, rs.hn, rs.chunks, rs.n_heavy, rs.n_chunks, 0};
            const ExArgs ua{rs.rp, rs.col, rs.tiles, rs.order, kb->dirs[usw].ulist, rs.hrank, nullptr, nullptr,
                            kb->dirs[usw].UW4};
            if (rs.n_chunks) {
                prof_begin(s, KC_SLICE_HEAVY);
                if (cls == 0) k_slice_heavy<false, 2><<<dim3(rs.n_chunks, packs), 256, 0, s>>>(su, sc, dd, run);
                else k_slice_heavy<true, 2><<<dim3(rs.n_chunks, packs), 256, 0, s>>>(su, sc, dd, run);
                count_launch();
                prof_end(s, KC_SLICE_HEAVY, 36.0 * rs.E_heavy * packs, 32.0 * rs.E_heavy * packs);
            }
            if (rs.n_blocks) {
                prof_begin(s, KC_SLICE_U);
                if (cls == 0) k_slice_ex<false><<<dim3(rs.n_blocks, packs), 256, 0, s>>>(ua, sc, dd, run, counts);
                else k_slice_ex<true><<<dim3(rs.n_blocks, packs), 256, 0, s>>>(ua, sc, dd, run, counts);
                count_launch();
                prof_end(s, KC_SLICE_U, (8.0 * rs.n_rows + 36.0 * rs.E) * packs + 4.0 * kb->dirs[usw].UW * run, 32.0 * rs.E * packs);
            }
            off += run;
            continue;
        }
        const SliceDir &hd = ex ? sdx : sd;
        if (hd.n_chunks) {
            prof_begin(s, KC_SLICE_HEAVY);
            if (pair) {
                if (cls == 0) k_slice_heavy<false, 4><<<dim3(hd.n_chunks, 1), 256, 0, s>>>(hd, sc, dd, run);
                else k_slice_heavy<true, 4><<<dim3(hd.n_chunks, 1), 256, 0, s>>>(hd, sc, dd, run);
            } else if (narrow) {
                if (cls == 0) k_slice_heavy<false, 1><<<dim3(hd.n_chunks, 1), 256, 0, s>>>(hd, sc, dd, run);
                else k_slice_heavy<true, 1><<<dim3(hd.n_chunks, 1), 256, 0, s>>>(hd, sc, dd, run);
            } else {
                if (cls == 0) k_slice_heavy<false, 2><<<dim3(hd.n_chunks, packs), 256, 0, s>>>(hd, sc, dd, run);
                else k_slice_heavy<true, 2><<<dim3(hd.n_chunks, packs), 256, 0, s>>>(hd, sc, dd, run);
            }
            count_launch();
            const double eh = ex ? (double)dr.E_ex_heavy : (double)dr.E_heavy;
            const double hb = narrow ? 16.0 : 32.0;
            prof_end(s, KC_SLICE_HEAVY, 4.0 * eh * (pair ? 1 : packs) + hb * eh * packs, hb * eh * packs);   // a pair: one CSR pass
        }
        if (ex) {
            prof_begin(s, KC_SLICE_EX);
            if (cls == 0) k_slice_ex<false><<<dim3(dr.n_ex_blocks, packs), 256, 0, s>>>(xa, sc, dd, run, counts);
            else k_slice_ex<true><<<dim3(dr.n_ex_blocks, packs), 256, 0, s>>>(xa, sc, dd, run, counts);
            count_launch();
            // example rows only: their CSR rows + 32 B T gathers + the projected rows
            prof_end(s, KC_SLICE_EX, (8.0 * kb->M + 36.0 * dr.E_ex) * packs + 4.0 * kb->MW * run, 32.0 * dr.E_ex * packs);
        } else {
            prof_begin(s, KC_SLICE);
            if (timing_enabled())
                std::fprintf(stderr, "[hedl slice] full sweep: dir %u class %u nodes %u%s\n", dirid, cls, run,
                             pair ? " (pair)" : narrow ? " (narrow)" : "");
#ifdef HEDL_DEBUG_TILE
            // timing experiments only (tools/dbg_tile.sh): skips sweep phases, results are WRONG
            static const uint32_t dbg = getenv("HEDL_DBG_TILE") ? (uint32_t)atoi(getenv("HEDL_DBG_TILE")) : 0u;
#else
            constexpr uint32_t dbg = 0u;
#endif
            // persistent grid: every resident CTA slot once (the tiles are taken dynamically);
            // occupancy per device (the carveout above is set per device)
            static std::once_flag occ_once[kMaxDevices];
            static uint32_t occ[kMaxDevices][6];
            int cur = 0;
            cudaGetDevice(&cur);
            once_per_device(occ_once, [&] {
                int b[6] = {0, 0, 0, 0, 0, 0};
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[0], k_slice_tile<false, 2>, 256, smem);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[1], k_slice_tile<true, 2>, 256, smem);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[2], k_slice_tile<false, 4>, 512, smem2);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[3], k_slice_tile<true, 4>, 512, smem2);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[4], k_slice_tile<false, 1>, 256, smem1);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[5], k_slice_tile<true, 1>, 256, smem1);
                for (int i = 0; i < 6; ++i) occ[(unsigned)cur % kMaxDevices][i] = (uint32_t)std::max(1, b[i]);
            });
            const uint32_t oi = (pair ? 2u : narrow ? 4u : 0u) + (cls == 0 ? 0u : 1u);
            const uint32_t resident = occ[(unsigned)cur % kMaxDevices][oi] * std::max(1, kb->sm_count);
            uint32_t *sched = (uint32_t *)(base + need - 256);   // self-cleaning {next tile, CTAs done}
            const uint32_t grid = std::min(dr.n_tiles, resident);
            UTab ut{};
            uint32_t uw4max = 0;
            for (const hedl_dir &x : kb->dirs) uw4max = std::max(uw4max, x.UW4);
            ut.stride = uw4max;
            for (uint32_t q = 0; q < kMaxUDirs && q < kb->dirs.size(); ++q) {
                ut.um[q] = kb->dirs[q].ex_umask;
                ut.ub[q] = kb->dirs[q].ex_ubase;
                ut.nu[q] = kb->dirs[q].n_u;
                ut.ul[q] = kb->dirs[q].ulist;
            }
            if (pair) {
                if (cls == 0) k_slice_tile<false, 4><<<grid, 512, smem2, s>>>(kd, sd, sc, ut, dd, run, counts, sched, dbg);
                else k_slice_tile<true, 4><<<grid, 512, smem2, s>>>(kd, sd, sc, ut, dd, run, counts, sched, dbg);
            } else if (narrow) {
                if (cls == 0) k_slice_tile<false, 1><<<grid, 256, smem1, s>>>(kd, sd, sc, ut, dd, run, counts, sched, dbg);
                else k_slice_tile<true, 1><<<grid, 256, smem1, s>>>(kd, sd, sc, ut, dd, run, counts, sched, dbg);
            } else {
                if (cls == 0) k_slice_tile<false, 2><<<grid, 256, smem, s>>>(kd, sd, sc, ut, dd, run, counts, sched, dbg);
                else k_slice_tile<true, 2><<<grid, 256, smem, s>>>(kd, sd, sc, ut, dd, run, counts, sched, dbg);
            }
            count_launch();
            // minimal DRAM bytes of one lane-packed pass: CSR once + T once (32 B per individual)
            // + the output rows; the 32 B-per-edge T gathers are L2 traffic (DESIGN.md K-SLICE)
            const double rb = narrow ? 16.0 : 32.0;       // T record bytes per pack
            prof_end(s, KC_SLICE, csr + rb * 32 * kb->W4 * packs + 4.0 * kb->W * run, rb * (double)(dr.E - dr.E_heavy) * packs);
        }
        off += run;
    }
    return HEDL_OK;
}

}  // namespace hedl

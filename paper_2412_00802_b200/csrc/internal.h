// Internal definitions of the hedl library (not part of the ABI).
// Device layout of the knowledge base: SURVEY 8(a) row a0 / DESIGN.md "Data layout".
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/hedl.h"

namespace hedl {

// allocator that default-initialises (no zero fill) trivially constructible elements:
// large planning arrays are written in parallel right after allocation
template <class T>
struct NoInitAlloc : std::allocator<T> {
    template <class U> struct rebind { using other = NoInitAlloc<U>; };
    NoInitAlloc() = default;
    template <class U> NoInitAlloc(const NoInitAlloc<U> &) {}
    template <class U> void construct(U *p) { ::new ((void *)p) U; }
    template <class U, class... A> void construct(U *p, A &&...a) { ::new ((void *)p) U(std::forward<A>(a)...); }
};

// ---- degree bins ------------------------------------------
// light  : deg <= kLightDeg      lane = individual, ballot builds the word
// medium : deg <= kHeavyDeg      warp-cooperative, 32 neighbours per step
// heavy  : deg >  kHeavyDeg      CTA chunks of kHeavyChunk edges, atomics + last-CTA finalise
constexpr uint32_t kLightDeg = 32;
constexpr uint32_t kHeavyDeg = 512;
constexpr uint32_t kMidDeg = 128;     // lane-packed sweep: medium rows up to this degree go 4 per warp
#ifndef HEDL_HEAVY_CHUNK
#define HEDL_HEAVY_CHUNK 4096
#endif
constexpr uint32_t kHeavyChunk = HEDL_HEAVY_CHUNK;
// a direction's heavy-row chunk: half size when the full-size chunks would not give four
// CTAs per SM (C4: 2.2M heavy edges per direction, 537 chunks of 4,096 on 148 SMs) --
// measured: C4 heavy-row sweeps 1.50 -> 1.39 ms per step, C5 (enough chunks) unchanged
inline uint32_t heavy_chunk(uint64_t heavy_edges, int sm_count) {
    return heavy_edges >= (uint64_t)kHeavyChunk * 4u * (uint64_t)(sm_count > 0 ? sm_count : 148) ? kHeavyChunk
                                                                                                  : kHeavyChunk / 2;
}
constexpr uint32_t kTopKMax = 4096;       // hedl_score_topk: k <= this
constexpr uint32_t kMaxUDirs = 4;         // role directions whose U rows restrictions can emit / U sweeps

// ---- restriction predicates ---------------------------------------------------
// Every role restriction counts the neighbours y of x whose (possibly
// complemented) child bit is 1, saturating at `sat`, then applies `pred`:
//   EXISTS  : count C,      GE n=1   (Alg. 4: a matching assertion sets x)
//   FORALL  : count not-C,  LE n=0   (Alg. 6: a non-matching assertion clears x)
//   MIN/MAX/EXACT: count C, GE / LE / EQ n  (Alg. 7-8), LEP = paper MAX
enum Pred : uint8_t { P_GE = 0, P_LE = 1, P_EQ = 2, P_LEP = 3 };

// ---- canonical program ---------------------------------------------------------
// Operand reference: bit0 = complement, bits1-2 = type, bits 3.. = id.
enum RefType : uint32_t { RT_NODE = 0, RT_ATOM = 1, RT_TOP = 2 };
inline uint32_t mkref(RefType t, uint32_t id, uint32_t comp) { return (id << 3) | (uint32_t(t) << 1) | comp; }
inline uint32_t ref_comp(uint32_t r) { return r & 1u; }
inline RefType ref_type(uint32_t r) { return RefType((r >> 1) & 3u); }
inline uint32_t ref_id(uint32_t r) { return r >> 3; }

enum NodeKind : uint8_t { NK_AND = 0, NK_OR = 1, NK_RESTRICT = 2, NK_DRANGE = 3, NK_STRING = 4 };
enum StrMode : uint8_t { SM_EQUAL = 0, SM_CONTAIN = 1 };

struct CNode {
    uint8_t kind;        // NodeKind
    uint8_t pred;        // restrict: Pred ; string: StrMode
    uint16_t dir;        // restrict: 2*role + inverse ; drange: data property ; string: string role
    uint32_t n;          // restrict: threshold ; string: interned value id (EQUAL) / program pattern id (CONTAIN)
    uint32_t sat;        // restrict: saturation point of the count
    float lo, hi;        // drange
    uint32_t op_begin;   // operands in Program::ops
    uint32_t op_count;   // AND/OR: k ; RESTRICT: 1 (child, complement already folded) ; DRANGE: 0
    uint32_t level;      // 1 + max level of node operands (0 if none)
    double bytes;        // algorithmic bytes of this node
};

}  // namespace hedl

// ---- handles -------------------------------------------------------------------
// a row subset of one direction's CSR, in the layout of the example-row (EX) sweep: rows
// ("ranks") in blocks of 128, medium then light rows per block by degree, heavy rows in
// 4,096-edge chunks, neighbours as individual ids
struct hedl_rowset {
    uint32_t n_rows = 0, n_blocks = 0, n_heavy = 0, n_chunks = 0;
    uint64_t E = 0, E_heavy = 0;
    double frac = 1.0;                             // (E + E_heavy) / the direction's E: sweep cost ratio
    uint32_t *rp = nullptr, *col = nullptr;        // device [n_rows+1], [E + E_heavy]
    uint4 *tiles = nullptr;                        // device [n_blocks+1] {order begin, n_med, n_light, heavy begin}
    uint32_t *order = nullptr, *hx = nullptr, *hrank = nullptr, *hn = nullptr;
    uint4 *chunks = nullptr;
};

struct hedl_dir {                  // one role direction
    uint32_t *row_ptr = nullptr;   // device [N+1]
    uint32_t *col = nullptr;       // device [E], sorted per row
    uint64_t E = 0;
    uint32_t n_heavy = 0, n_chunks = 0;
    uint32_t *heavy_x = nullptr;       // device [n_heavy]
    uint32_t *heavy_nchunks = nullptr; // device [n_heavy]
    uint4 *chunks = nullptr;           // device [n_chunks] {heavy idx, e0, e1, 0}
    std::vector<uint32_t> h_row_ptr;   // host copy (planning of lane-packed kernels)
    uint32_t max_deg = 0;
    uint64_t E_heavy = 0;              // edges of heavy rows
    // lane-packed path: per 1024-individual tile {order begin, n_medium, n_light, heavy begin}
    uint32_t n_tiles = 0;
    uint4 *tiles = nullptr;            // device [n_tiles + 1]
    uint32_t *order = nullptr;         // device [N - n_heavy]: per tile medium rows then light rows, degree-descending
    uint32_t *tile_rank = nullptr;     // device [n_tiles]: tiles in decreasing sweep cost (persistent scheduling)
    uint32_t *tile_nbig = nullptr;     // device [n_tiles]: medium rows of the tile with deg > kMidDeg
    // light rows of each tile in SELL-16 slices (16 rows of similar degree, neighbours interleaved
    // so the 16 row-pairs of a warp read 16 consecutive indices per step; pads = 0xffffffff)
    uint32_t *tile_slice = nullptr;    // device [n_tiles + 1]: first slice of each tile
    uint32_t *sell_off = nullptr;      // device [n_slices]: offset into sell_col
    uint32_t *sell_w = nullptr;        // device [n_slices]: width (max degree) of the slice
    uint32_t *sell_col = nullptr;      // device
    // example-row ("EX") packs: the same over the example ranks, 128 ranks per block
    uint32_t n_ex_blocks = 0;
    uint4 *ex_tiles = nullptr;         // device [n_ex_blocks + 1] {order begin, n_medium, n_light, ex-heavy begin}
    uint32_t *ex_order = nullptr;      // device: example ranks (medium then light, degree-descending per block)
    uint32_t n_ex_heavy = 0, n_ex_chunks = 0;
    uint32_t *ex_hx = nullptr, *ex_hrank = nullptr, *ex_hn = nullptr;   // heavy example rows: id, rank, #chunks
    uint4 *ex_chunks = nullptr;        // {ex-heavy idx, e0, e1, 0}
    uint64_t E_ex = 0, E_ex_heavy = 0; // edges of light/medium and of heavy example rows
    // compact T for EX packs: U = sorted distinct neighbours of the example rows; an EX pack
    // stores T only at U (32 B each) and the example rows' edges point into it
    uint32_t n_u = 0;
    uint32_t *ex_rp = nullptr;         // device [M+1]: edge range of example rank r
    uint32_t *ex_ccol = nullptr;       // device: compact T index of each such edge's neighbour
    uint32_t *ex_umask = nullptr;      // device [W4]: bit y&31 of word y>>5 set iff y in U
    uint32_t *ex_ubase = nullptr;      // device [W4]: |U ∩ [0, 32w)|
    // U-space rows: a row over U (bit t = individual U[t]),
    // UW4 words (padded to 8); the fillers of EX-pack restrictions are evaluated / stored here
    uint32_t UW = 0, UW4 = 0;
    uint32_t *uconcepts = nullptr;     // device [C][UW4]
    uint32_t *uones = nullptr;         // device [UW4], tail-masked TOP row over U
    uint32_t *ulist = nullptr;         // device [n_u]: the members of U in order (U position -> individual)
    // U sweeps: this direction's rows restricted to U_d' (for restrictions needed only over
    // one U_d'), per d' < kMaxUDirs (empty without examples or with more directions)
    hedl_rowset usw[hedl::kMaxUDirs];
};

struct hedl_data {
    uint32_t *row_ptr = nullptr;   // device [N+1]
    float *val = nullptr;          // device [V], ascending within each individual
    uint64_t V = 0;
};

struct hedl_sdir {                 // one string concrete role (Algs. 11-14)
    uint32_t *row_ptr = nullptr;   // device [N+1]: subject -> its distinct value ids
    uint32_t *vid = nullptr;       // device [E], ascending per subject
    uint64_t *dict_off = nullptr;  // device [V+1]: interned value v = dict[dict_off[v] .. dict_off[v+1])
    uint8_t *dict = nullptr;       // device
    uint64_t E = 0, V = 0, dict_bytes = 0;
    std::unordered_map<std::string, uint32_t> ids;   // host: value -> id (stringValuesMapping)
};

struct hedl_kb {
    int device = 0;
    int sm_count = 148;
    uint32_t N = 0, W = 0, W4 = 0, C = 0, R = 0, D = 0;
    uint32_t *concepts = nullptr;  // device [C][W4]
    uint32_t *ones = nullptr;      // device [W4], tail-masked TOP row
    uint32_t *zeros = nullptr;     // device [W4]
    uint32_t *pos = nullptr, *neg = nullptr;  // device [W4]
    uint64_t npos = 0, nneg = 0;
    // example projection: E = sorted P u N, M = |E|;
    // a projected row holds bit r = membership of the r-th example (MW4 = ceil(M/32) padded to 4)
    uint32_t M = 0, MW = 0, MW4 = 0;
    uint32_t *ex_mask = nullptr, *ex_base = nullptr;    // device [W4]
    uint32_t *ex_ids = nullptr;                         // device [M]: the examples in rank order
    std::vector<uint32_t> h_ex;                         // host copy of ex_ids
    uint32_t *pconcepts = nullptr;                      // device [C][MW4]
    uint32_t *pones = nullptr, *ppos = nullptr, *pneg = nullptr;   // device [MW4]
    std::vector<hedl_dir> dirs;    // 2R
    std::vector<hedl_data> data;   // D
    uint32_t S = 0;
    std::vector<hedl_sdir> sdirs;  // S string roles
    std::vector<void *> allocs;
    uint64_t device_bytes = 0;
    std::atomic<bool> poisoned{false};
    std::atomic<int> refs{1};            // the handle itself + every live program compiled against it
    // buffers released by freed programs, reused by the next ones (no cudaMalloc /
    // cudaMallocHost / memset per program); accumulator buffers return self-cleaned
    mutable std::mutex pool_mu;
    mutable std::vector<std::pair<void *, size_t>> pool[16];
    const void **interp_ptrs = nullptr;  // device: per-direction row_ptr/col, per-property row_ptr/val
    std::mutex interp_mu;
    std::vector<double> dir_bytes;  // 4(N+1) + 4E per direction
    std::vector<double> data_bytes; // 4(N+1) + 4V per property
    std::vector<double> str_bytes;  // 4(N+1) + 4E (+ dictionary for CONTAIN) per string role
};

struct hedl_program {
    const hedl_kb *kb = nullptr;
    uint32_t flags = 0;
    std::vector<hedl::CNode, hedl::NoInitAlloc<hedl::CNode>> nodes;
    std::vector<uint32_t, hedl::NoInitAlloc<uint32_t>> ops;
    std::vector<uint32_t> root_node;   // per root: computed canonical node id
    std::vector<std::string> patterns; // CONTAIN patterns (deduplicated), CNode.n indexes them
    std::vector<double> root_bytes;    // B(h)
    uint32_t n_levels = 0;
    // evaluation workspace (device), grown on demand
    std::mutex mu;
    void *ws = nullptr;
    size_t ws_bytes = 0;
    void *pinned = nullptr;
    size_t pinned_bytes = 0;
    uint64_t ws_limit = 0;              // 0 = auto (half the free memory, <= 48 GiB)
    // latency path: mapped pinned counts (host pointer + device alias)
    hedl_counts *lat_host = nullptr, *lat_dev = nullptr;   // [2]: counts, completion sequence
    uint64_t lat_seq = 0;
    // planning scratch (host)
    std::vector<uint32_t> stamp;
    uint32_t stamp_gen = 0;
    // device-compiled program (hedl_compile_device): canonical DAG in device memory
    bool dev = false, dev_downloaded = false;
    hedl::CNode *d_nodes = nullptr;
    uint32_t *d_ops = nullptr, *d_root_node = nullptr;
    void *d_block = nullptr;            // the pooled block holding the three arrays
    size_t d_block_bytes = 0;
    uint32_t dev_n_nodes = 0, dev_n_roots = 0;
    uint64_t dev_n_ops = 0;
    void *dplan = nullptr;              // device-side evaluation plan state (dplan.cu)
};

namespace hedl {

// ---- device-compiled programs (dcompile.cu) ---------------------------------------
void dc_free_arrays(hedl_program *p);
hedl_status dc_download(hedl_program *p);     // host copy of nodes / ops / roots (utilities)
inline uint32_t prog_n_roots(const hedl_program *p) { return p->dev ? p->dev_n_roots : (uint32_t)p->root_node.size(); }

// ---- errors --------------------------------------------------------------------
void set_error(const std::string &msg);
hedl_status fail(hedl_status st, const std::string &msg);
hedl_status cuda_fail(const hedl_kb *kb, cudaError_t e, const char *where);

#define HEDL_CUDA(kb, call)                                  \
    do {                                                     \
        cudaError_t _e = (call);                             \
        if (_e != cudaSuccess) return hedl::cuda_fail(kb, _e, #call); \
    } while (0)

// ---- workspace pool (per KB) ---------------------------------------------------
enum PoolRole { PR_ROWS, PR_PROWS, PR_HEAVY, PR_COUNTS, PR_SLICE, PR_PLAN_DEV, PR_PLAN_HOST, PR_DC_SCRATCH, PR_DC_PROG,
                PR_DPLAN, PR_DPLAN_HOST, PR_UROWS, PR_N };
void *pool_take(const hedl_kb *kb, int role, size_t need, size_t *got);
void pool_give(const hedl_kb *kb, int role, void *p, size_t bytes);
void pool_release_all(hedl_kb *kb);
// device memory: the caller's allocator (hedl_set_allocator) or cudaMalloc / cudaFree
cudaError_t dev_malloc(void **p, size_t bytes, cudaStream_t s = nullptr);
void dev_free(void *p, cudaStream_t s = nullptr);
bool dev_alloc_installed();
void live_kb_add(int d);                   // KBs alive (the allocator may change only at 0)
// a device block from the pool (best fit) or dev_malloc (25% headroom); null on OOM
inline void *pool_alloc(const hedl_kb *kb, int role, size_t need, size_t *got) {
    if (void *q = pool_take(kb, role, need, got)) return q;
    void *q = nullptr;
    const size_t sz = (need * 5 / 4 + 255) & ~size_t(255);
    if (dev_malloc(&q, sz) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    *got = sz;
    return q;
}
// carves aligned sub-arrays out of one block (base == null: sizing pass)
struct Carver {
    char *base = nullptr;
    size_t off = 0;
    template <class T> T *take(size_t n) {
        off = (off + 255) & ~size_t(255);
        T *r = base ? (T *)(base + off) : nullptr;
        off += std::max<size_t>(n * sizeof(T), 16);
        return r;
    }
};
void kb_release(const hedl_kb *kb);     // drop one reference; frees the KB at zero

// Function attributes (dynamic shared memory opt-in, carveout) belong to a device's
// context, and KBs may live on any device of the process: run `f` once per device,
// thread-safe.  Each call site owns its flag array.
constexpr int kMaxDevices = 64;
template <class F>
inline void once_per_device(std::once_flag (&flags)[kMaxDevices], F f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(flags[(unsigned)dev % kMaxDevices], f);
}

// ---- host phase timing (HEDL_TIMING=1 prints to stderr) ---------------------------
bool timing_enabled();
double now_ms();
void timing_note(const char *what, double ms);

// ---- profiling -----------------------------------------------------------------
enum KClass { KC_BOOL, KC_RESTRICT, KC_HEAVY, KC_DRANGE, KC_COVER_INIT, KC_GATHER,
              KC_SLICE_IN, KC_SLICE, KC_SLICE_HEAVY, KC_KB, KC_SLICE_EX, KC_INTERP, KC_STRING, KC_BOOL_L2, KC_SLICE_U, KC_N };
extern const char *kKClassName[KC_N];
void prof_begin(cudaStream_t s, int kc);
bool prof_active();
void prof_end(cudaStream_t s, int kc, double alg_bytes, double units = 1);

// ---- kernels launchers (kernels.cu) -----------------------------------------
struct BoolDesc {
    uint32_t *out;
    uint32_t *proj;                // example-projected copy of the output (null = not needed)
    uint32_t op_first, op_count;   // into the operand table
    uint32_t is_or;
    int32_t cover;                 // counts slot or -1
};
struct Operand {
    const uint32_t *ptr;
    uint32_t mask;                 // 0 or ~0 (complement)
    uint32_t pad;
};
struct RestrictDesc {
    const uint32_t *child;
    uint32_t *out;
    uint32_t *proj;                // example-projected copy of the output (null = not needed)
    uint32_t cmask;                // 0 or ~0
    uint32_t pred, n, sat;
    int32_t cover;                 // counts slot or -1
    uint32_t heavy_slot;           // scratch base index for heavy counters of this node
    // fused filler (lane packs only; child == null): the filler is the AND (OR if bit 31 of
    // op_n) of operands [op_first, op_first + (op_n & 0x7fffffff)) of the plan's operand table
    uint32_t op_first, op_n;
    // U rows this restriction emits from its full-pack epilogue (DESIGN.md "U rows of
    // restrictions"): direction d (bit d of udirs, d < kMaxUDirs) -> uout + rank of d in udirs
    // x the U-row stride; zeroed before the chunk, filled with atomicOr
    uint32_t *uout;
    uint32_t udirs, pad_;
};

constexpr uint32_t kFuseMaxOps = 4;   // operands of a boolean filler the pack kernel combines
struct DrangeDesc {
    uint32_t *out;
    uint32_t *proj;
    float lo, hi;
    int32_t cover;
    uint32_t prop;
};
struct StringDesc {
    uint32_t *out;
    uint32_t *proj;
    int32_t cover;
    uint32_t mode;                 // StrMode
    uint32_t vid;                  // EQUAL: interned value id
    uint32_t pat_len;              // CONTAIN: pattern bytes pat[0 .. pat_len)
    const uint8_t *pat;            // device (the plan's pattern blob)
};
struct StrDev {                   // one string role, passed by value
    const uint32_t *row_ptr, *vid;
    const uint64_t *dict_off;
    const uint8_t *dict;
};
struct DirDev {                   // passed by value
    const uint32_t *row_ptr;
    const uint32_t *col;
    const uint32_t *heavy_x;
    const uint32_t *heavy_nchunks;
    const uint4 *chunks;
    uint32_t n_heavy, n_chunks;
    const uint4 *tiles;             // per-tile row order (medium, light) and SELL-16 light slices
    const uint32_t *order, *tile_slice, *sell_off, *sell_w, *sell_col;
    uint32_t n_tiles;
};
struct KbDev {
    uint32_t N, W, W4;
    const uint32_t *pos, *neg;
    const uint32_t *ex_mask, *ex_base;   // example projection: per word, example bits and rank of the first
};

#ifdef __CUDACC__
// Checked build (-DHEDL_CHECKED, tools/checked.sh): device-side bounds / invariant traps in the
// hot kernels and guard zones around every device block (api.cpp).  Compiled out otherwise.
#ifdef HEDL_CHECKED
#define HCHECK(c)                                                                                 \
    do {                                                                                          \
        if (!(c)) {                                                                               \
            printf("HCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, \
                   threadIdx.x, #c);                                                              \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define HCHECK(c) ((void)0)
#endif
#endif

#ifdef __CUDACC__
// scatter the example bits of full-row word w into an example-projected row (atomicOr;
// the projected row is zeroed before the launch)
static __device__ __forceinline__ void proj_scatter(const KbDev &kb, uint32_t *proj, uint32_t w, uint32_t word) {
    uint32_t m = __ldg(kb.ex_mask + w);
    if (!m || !word) return;
    uint32_t bits = 0, nb = 0;
    for (; m; m &= m - 1, ++nb) bits |= ((word >> (__ffs(m) - 1)) & 1u) << nb;   // pext(word, mask)
    if (!bits) return;
    const uint32_t base = __ldg(kb.ex_base + w), sh = base & 31;
    atomicOr(proj + (base >> 5), bits << sh);
    if (sh && sh + nb > 32) atomicOr(proj + (base >> 5) + 1, bits >> (32 - sh));
}
#endif
void launch_cover_init(cudaStream_t s, hedl_counts *counts, uint32_t n, uint64_t npos, uint64_t nneg);
void launch_bool(cudaStream_t s, const KbDev &kb, const BoolDesc *d_desc, uint32_t n_desc,
                 const Operand *d_ops, hedl_counts *counts, double alg_bytes, uint64_t npos, uint64_t nneg,
                 bool full_rows);
// inv / push (nullable): the inverse direction and self-cleaning scratch of push_stride words
// per node -- groups of <= kPushMaxNodes nodes then pick push or pull per node on the device
void launch_restrict(cudaStream_t s, const KbDev &kb, const DirDev &dir, const RestrictDesc *d_desc,
                     uint32_t n_desc, hedl_counts *counts, uint32_t *heavy_scratch, double alg_light,
                     double alg_heavy, const DirDev *inv = nullptr, uint32_t *push = nullptr, size_t push_stride = 0);
constexpr uint32_t kPushMaxNodes = 8;      // per-node groups this small consider the push direction
constexpr uint32_t kPushMinN = 1u << 18;   // ... on KBs at least this large (below, the pull is cheap)
size_t push_scratch_words(uint32_t N, uint32_t W4, bool counting);
// xmap != null: U space of a direction (kb = {|U|, UW, UW4}); position p is individual xmap[p]
void launch_drange(cudaStream_t s, const KbDev &kb, const uint32_t *row_ptr, const float *val,
                   const DrangeDesc *d_desc, uint32_t n_desc, hedl_counts *counts, double alg_bytes,
                   const uint32_t *xmap = nullptr);
void launch_string(cudaStream_t s, const KbDev &kb, const StrDev &sd, const StringDesc *d_desc, uint32_t n_desc,
                   hedl_counts *counts, double alg_bytes);
void launch_gather_counts(cudaStream_t s, const hedl_counts *slots, const uint32_t *slot_of,
                          hedl_counts *out, uint32_t n);
void launch_gather_bits(cudaStream_t s, const uint32_t *const *rows, uint32_t *out, uint32_t W,
                        uint32_t n);
void launch_kb_build(cudaStream_t s);
uint64_t launches_total();
void count_launch();
void count_launches(uint64_t n);
void count_io(uint64_t h2d, uint64_t d2h);

}  // namespace hedl

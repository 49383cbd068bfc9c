// Rows supplied by the caller (one hypothesis split across GPUs).
//
// In the individual-range partition (paper_2412_00802_b200/dist.py eval_split), each rank
// evaluates every node only for the individuals it owns, and a restriction's filler must be
// complete before the restriction runs: the ranks all_gather their word segments of the
// filler rows and write the complete rows into reserved ("scratch") concept slots of their
// KB with hedl_kb_set_concept_rows.  The filler is then an ordinary atomic concept of the
// restriction -- the per-level exchange step of PAPER.md:563-578's multi-device scheduling,
// with the paper's "exact copy of knowledge representation matrixes" replaced
// by a partition of the assertions.
//
// A concept row has derived copies the planner reads instead of the full row: its
// example-projected row (bit r = the r-th example) and, per
// role direction, its U row (bit t = the t-th neighbour of an example, "U-projected rows").
// Both are rebuilt here from the new row with the same masks the loader used.
#include "internal.h"

using namespace hedl;

namespace {

// dst row i (W4 words) = concatenation over p of src[p][i][0 .. part_words), truncated to W
// words, tail bits above N cleared, padding words zero
__global__ void k_assemble_rows(const uint32_t *__restrict__ src, uint32_t n, uint32_t parts, uint32_t part_words,
                                uint32_t *__restrict__ dst, uint32_t N, uint32_t W, uint32_t W4) {
    const uint64_t total = (uint64_t)n * W4;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(k / W4), w = (uint32_t)(k % W4);
        uint32_t v = 0;
        if (w < W) {
            const uint32_t p = w / part_words, o = w % part_words;
            v = p < parts ? __ldg(src + ((uint64_t)p * n + i) * part_words + o) : 0u;
            if (w == W - 1 && (N & 31)) v &= (1u << (N & 31)) - 1u;
        }
        dst[(uint64_t)i * W4 + w] = v;
    }
}

// projected rows: for every word w of row i, the bits at `mask[w]` (pext) go to bit positions
// base[w] .. of the projected row (dst zeroed before the launch; atomicOr at word seams)
__global__ void k_project_rows(const uint32_t *__restrict__ rows, uint32_t n, uint32_t W4,
                               const uint32_t *__restrict__ mask, const uint32_t *__restrict__ base,
                               uint32_t *__restrict__ dst, uint32_t dst_w4) {
    const uint64_t total = (uint64_t)n * W4;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(k / W4), w = (uint32_t)(k % W4);
        uint32_t m = __ldg(mask + w);
        const uint32_t word = __ldg(rows + k);
        if (!m || !word) continue;
        uint32_t bits = 0, nb = 0;
        for (; m; m &= m - 1, ++nb) bits |= ((word >> (__ffs(m) - 1)) & 1u) << nb;
        if (!bits) continue;
        const uint32_t b = __ldg(base + w), sh = b & 31;
        uint32_t *d = dst + (uint64_t)i * dst_w4 + (b >> 5);
        atomicOr(d, bits << sh);
        if (sh && sh + nb > 32) atomicOr(d + 1, bits >> (32 - sh));
    }
}

inline uint32_t grid_for(uint64_t work) {
    const uint64_t b = (work + 255) / 256;
    return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 16));
}

}  // namespace

extern "C" hedl_status hedl_kb_set_concept_rows(hedl_kb *kb, uint32_t first, uint32_t n, const uint32_t *src,
                                                uint32_t parts, uint32_t part_words, void *stream) {
    if (!kb) return fail(HEDL_ERR_INVALID_ARG, "null kb");
    if (kb->poisoned) return fail(HEDL_ERR_CUDA, "KB handle is poisoned by an earlier CUDA error");
    if ((uint64_t)first + n > kb->C) return fail(HEDL_ERR_OUT_OF_RANGE, "concept range out of range");
    if (!n || !kb->W) return HEDL_OK;
    if (!src || !parts || !part_words) return fail(HEDL_ERR_INVALID_ARG, "null src or zero parts / part_words");
    if ((uint64_t)parts * part_words < kb->W) return fail(HEDL_ERR_INVALID_ARG, "parts x part_words < row words");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != kb->device) cudaSetDevice(kb->device);
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *rows = kb->concepts + (uint64_t)first * kb->W4;
    prof_begin(s, KC_KB);
    k_assemble_rows<<<grid_for((uint64_t)n * kb->W4), 256, 0, s>>>(src, n, parts, part_words, rows, kb->N, kb->W, kb->W4);
    count_launch();
    if (kb->MW4) {
        uint32_t *pr = kb->pconcepts + (uint64_t)first * kb->MW4;
        HEDL_CUDA(kb, cudaMemsetAsync(pr, 0, (size_t)n * kb->MW4 * 4, s));
        k_project_rows<<<grid_for((uint64_t)n * kb->W4), 256, 0, s>>>(rows, n, kb->W4, kb->ex_mask, kb->ex_base, pr, kb->MW4);
        count_launch();
    }
    for (const hedl_dir &d : kb->dirs) {
        if (!d.UW4 || !d.uconcepts) continue;
        uint32_t *ur = d.uconcepts + (uint64_t)first * d.UW4;
        HEDL_CUDA(kb, cudaMemsetAsync(ur, 0, (size_t)n * d.UW4 * 4, s));
        k_project_rows<<<grid_for((uint64_t)n * kb->W4), 256, 0, s>>>(rows, n, kb->W4, d.ex_umask, d.ex_ubase, ur, d.UW4);
        count_launch();
    }
    prof_end(s, KC_KB, 8.0 * n * kb->W4, n);
    HEDL_CUDA(kb, cudaGetLastError());
    return HEDL_OK;
}

/*
 * hedl.h -- C ABI of the B200-native HT-HEDL hot path (arxiv 2412.00802).
 *
 * The library evaluates ALCQI(D) concept hypotheses against an ABox under the
 * paper's closed-world / unique-name instance semantics (§III,
 * PAPER.md:53 §III-A) and counts covered positive/negative examples
 * (§IV Alg. 15).  Problem statement: "evaluate hypotheses up
 * to the ALCQI(D) DL language"; evaluation plan PAPER.md:532.
 *
 * Conventions
 *  - Every function returns hedl_status (HEDL_OK == 0).  On error no handle is
 *    created, outputs are unspecified, and hedl_last_error() returns a
 *    thread-local message naming the offending node / hypothesis index.  No C++
 *    exception crosses this boundary.
 *  - A bitset ("row") over the N individuals is W = ceil(N/32) uint32 words,
 *    LSB-first: individual i is bit (i & 31) of word (i >> 5).  Tail bits of the
 *    last word are 0 in every input, stored, returned or compared row
 *    (SURVEY Q6).  This replaces the paper's one byte per membership
 *    ("16 (8-bit) concept memberships").
 *  - "device" pointers are CUDA device addresses on the KB's device; "host"
 *    pointers are ordinary CPU memory.  Input arrays are borrowed for the call
 *    and copied; output buffers are owned by the caller.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Handles are opaque.  A hedl_kb is immutable after load and may be shared by
 *    concurrent evaluations.  A hedl_program owns a workspace; concurrent eval
 *    calls on ONE program serialise on an internal mutex (use one program per
 *    stream for concurrency).  A CUDA error poisons the KB handle: every later
 *    call on it returns HEDL_ERR_CUDA.
 */
#ifndef HEDL_H
#define HEDL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hedl_status;
#define HEDL_OK 0
#define HEDL_ERR_INVALID_ARG 1     /* null/ill-sized argument, non-zero tail bits, E >= 2^32 */
#define HEDL_ERR_OUT_OF_RANGE 2    /* an id >= its count (individual, concept, role, data, root) */
#define HEDL_ERR_EXAMPLE_CONFLICT 3 /* an individual is both positive and negative */
#define HEDL_ERR_BAD_EXPR 4        /* arity, cycle, NaN bound, n > 2^32-2, inverse data property */
#define HEDL_ERR_PARSE 5           /* hedl_compile_text: syntax error, unknown name, negative n */
#define HEDL_ERR_CUDA 6            /* CUDA runtime error; the KB handle is poisoned */
#define HEDL_ERR_OOM 7             /* host or device allocation failed */
#define HEDL_ERR_UNSUPPORTED 8     /* e.g. no sm_100 device */

typedef struct hedl_kb hedl_kb;
typedef struct hedl_program hedl_program;

/* ---------------------------------------------------------------------------
 * Knowledge base (§III-A, Fig. 3).  Fields:
 *   n_individuals  N; every individual id is < N.  N == 0 is legal (W == 0).
 *   n_concepts, concept_bits   host u32[C][W], row c = extension of concept c
 *                  (the transposed concepts matrix of PAPER.md:63, bit-packed).
 *   n_roles, role_edge_off     host u64[R+1]; role r's assertions are
 *                  (edge_subj[k], edge_obj[k]) for k in [off[r], off[r+1]).  Any
 *                  order; duplicates are removed (role extensions are sets,
 *                  SURVEY Q4).  Stored as CSR plus transposed CSR (r^-,
 *                  PAPER.md:299).  Each role must have < 2^32 distinct pairs.
 *   n_data, data_off, data_subj, data_val   numeric concrete roles
 *                  (§III-B3): assertions (data_subj[k], data_val[k])
 *                  for k in [data_off[d], data_off[d+1]); several values per
 *                  subject allowed; NaN values never match
 *                   and are dropped at load.
 *   pos_ids / neg_ids   host u32 lists of positive / negative examples
 *                  (ExMat); duplicates allowed; must be disjoint.
 *   n_strings, str_off, str_subj, str_val_off, str_bytes   string concrete
 *                  roles (PAPER.md:63 strConcretRoleMat, §III-B3 Algs. 11-14):
 *                  role s's assertions are k in [str_off[s], str_off[s+1]), host
 *                  u64[S+1]; assertion k is (str_subj[k], the byte string
 *                  str_bytes[str_val_off[k] .. str_val_off[k+1])), str_val_off
 *                  host u64[str_off[S]+1] ascending.  Values are raw bytes (no
 *                  terminator, may be empty, compared byte-wise).  Duplicate
 *                  (subject, value) pairs are removed; distinct values of a role
 *                  are interned (the paper's stringValuesMapping).
 *                  n_strings == 0 with null arrays is legal.
 * ------------------------------------------------------------------------- */
typedef struct hedl_kb_desc {
    uint32_t n_individuals;
    uint32_t n_concepts;
    const uint32_t *concept_bits;
    uint32_t n_roles;
    const uint64_t *role_edge_off;
    const uint32_t *edge_subj;
    const uint32_t *edge_obj;
    uint32_t n_data;
    const uint64_t *data_off;
    const uint32_t *data_subj;
    const float *data_val;
    uint32_t n_pos;
    const uint32_t *pos_ids;
    uint32_t n_neg;
    const uint32_t *neg_ids;
    uint32_t n_strings;
    const uint64_t *str_off;
    const uint32_t *str_subj;
    const uint64_t *str_val_off;
    const uint8_t *str_bytes;
} hedl_kb_desc;

typedef struct hedl_kb_info {
    uint32_t n_individuals, words, words_padded, n_concepts, n_roles, n_data;
    uint64_t n_pos, n_neg;
    uint64_t device_bytes;          /* bytes of device memory the KB holds */
    uint64_t edges[64];             /* distinct pairs per direction 2r (r) / 2r+1 (r^-), r < 32 */
    uint64_t heavy[64];             /* individuals above the heavy-degree threshold per direction */
    uint32_t n_strings;
    uint64_t str_pairs[32];         /* distinct (subject, value) pairs per string role, s < 32 */
    uint64_t str_values[32];        /* distinct values (interned strings) per string role */
} hedl_kb_info;

/* Build the device layout on `device` (copying through `stream`; returns after
 * the upload completed).  Errors: INVALID_ARG (null arrays with non-zero
 * counts, tail bits set, more than 32 roles / 65535 data properties / 65535
 * string roles / 2^29-1 concepts), OUT_OF_RANGE (id >= N), EXAMPLE_CONFLICT,
 * OOM, CUDA, UNSUPPORTED (device is not sm_100). */
hedl_status hedl_kb_load(const hedl_kb_desc *desc, int device, void *stream, hedl_kb **out);
hedl_status hedl_kb_free(hedl_kb *kb);
hedl_status hedl_kb_get_info(const hedl_kb *kb, hedl_kb_info *out);

/* Overwrite concept rows [first, first + n) with rows the caller supplies (SURVEY 8(f)
 * NEXT-4: one hypothesis split across GPUs by individual range; the
 * ranks all_gather their word segments of each restriction filler and install the
 * complete rows as "scratch" concepts reserved at load, see
 * paper_2412_00802_b200/dist.py eval_split).  src: DEVICE u32 [parts][n][part_words] --
 * row i is the concatenation over p of src[p][i][0 .. part_words), cut to W words
 * (parts * part_words >= W); bits above N are cleared.  The rows' derived copies
 * (example-projected and per-direction U rows) are rebuilt too.  Asynchronous on
 * `stream`.  This is the one call that mutates a KB: no evaluation on the KB may run
 * concurrently, and later evaluations on other streams must be ordered after it.
 * Errors: INVALID_ARG, OUT_OF_RANGE (first + n > n_concepts), CUDA. */
hedl_status hedl_kb_set_concept_rows(hedl_kb *kb, uint32_t first, uint32_t n, const uint32_t *src, uint32_t parts,
                                     uint32_t part_words, void *stream);

/* ---------------------------------------------------------------------------
 * Hypotheses (§IV: "a series of (potentially) nested DL
 * operations", stored contiguously; an "evaluation plan ... determines the
 * computational order").  A hypothesis batch is a node array; node i's
 * children are child_idx[child_begin .. child_begin+child_count).  Children
 * may be shared (a DAG is accepted); cycles are rejected.
 * ------------------------------------------------------------------------- */
#define HEDL_OP_TOP 0
#define HEDL_OP_BOTTOM 1
#define HEDL_OP_ATOM 2     /* arg = concept id */
#define HEDL_OP_NOT 3      /* 1 child; complement over Delta = {0..N-1} */
#define HEDL_OP_AND 4      /* k >= 0 children; empty AND = TOP (Alg. 1/2 "r=1")  */
#define HEDL_OP_OR 5       /* k >= 0 children; empty OR = BOTTOM ("=0 for disj.") */
#define HEDL_OP_EXISTS 6   /* arg = role; 1 child (Alg. 4)     */
#define HEDL_OP_FORALL 7   /* arg = role; 1 child (Alg. 6)     */
#define HEDL_OP_MIN 8      /* arg = role, n; >=n (Alg. 8 MIN)       */
#define HEDL_OP_MAX 9      /* arg = role, n; <=n, 0 included          */
#define HEDL_OP_EXACT 10   /* arg = role, n; ==n (Alg. 7 EXACTLY)   */
#define HEDL_OP_DRANGE 11  /* arg = data property; exists v in [lo,hi] (Alg. 10) */
#define HEDL_OP_SEQUAL 12  /* arg = string role, n = pattern id; exists value == pattern (Alg. 11-12) */
#define HEDL_OP_SCONTAIN 13 /* arg = string role, n = pattern id; exists value containing the
                              pattern as a contiguous byte substring (Alg. 13-14); the empty
                              pattern is rejected (BAD_EXPR, Q20) */

#define HEDL_FLAG_INV 1u   /* node.flags: the role is the inverse r^-  */

typedef struct hedl_node {
    uint8_t op;
    uint8_t flags;
    uint16_t reserved;      /* must be 0 */
    uint32_t arg;
    uint32_t n;             /* cardinality bound for MIN/MAX/EXACT (n <= 2^32-2); pattern id for SEQUAL/SCONTAIN */
    float lo, hi;           /* DRANGE closed float32 bounds; +-inf allowed, NaN rejected */
    uint32_t child_begin, child_count;
} hedl_node;

/* compile flags */
#define HEDL_COMPILE_NO_CSE 1u            /* do not merge identical subexpressions */
#define HEDL_COMPILE_NO_REWRITE 2u        /* no flatten / sort / dedupe of AND-OR operands */
#define HEDL_COMPILE_COMPAT_PAPER_MAX 4u  /* MAX as the paper's cVal>0 && cVal<=rVal */
#define HEDL_COMPILE_HOST_INPUT 8u        /* hedl_compile_device: the three input arrays are HOST memory */

/* Compile `roots` (indices into nodes) into a program: canonical DAG with
 * common-subexpression reuse across all roots, topological levels, per-node
 * algorithmic byte cost.  Host-only; `kb` supplies the id
 * bounds and sizes.  Errors: INVALID_ARG, OUT_OF_RANGE (child/root/arg id),
 * BAD_EXPR (arity, cycle, NaN bound, inverse data property, n > 2^32-2). */
hedl_status hedl_compile(const hedl_kb *kb, const hedl_node *nodes, uint32_t n_nodes,
                         const uint32_t *child_idx, uint64_t n_child_idx,
                         const uint32_t *roots, uint32_t n_roots, uint32_t flags,
                         hedl_program **out);
/* hedl_compile with a string-pattern table for SEQUAL / SCONTAIN nodes: pattern
 * p is the bytes pat_bytes[pat_off[p] .. pat_off[p+1]) (host u64[n_patterns+1],
 * ascending; copied).  SEQUAL resolves its pattern against the role's interned
 * values at compile time; a pattern no assertion holds compiles to BOTTOM with
 * no kernel work (the paper's short-circuit).  Errors as
 * hedl_compile, plus OUT_OF_RANGE (pattern id >= n_patterns, string role >=
 * n_strings) and BAD_EXPR (empty SCONTAIN pattern, children or INV flag on a
 * string node).  hedl_compile == hedl_compile_ex with no patterns. */
hedl_status hedl_compile_ex(const hedl_kb *kb, const hedl_node *nodes, uint32_t n_nodes,
                            const uint32_t *child_idx, uint64_t n_child_idx,
                            const uint32_t *roots, uint32_t n_roots, uint32_t flags,
                            uint32_t n_patterns, const uint64_t *pat_off, const uint8_t *pat_bytes,
                            hedl_program **out);
hedl_status hedl_program_free(hedl_program *prog);

/* Text front end (convenience and tests): SPEC.md:347-355's s-expression grammar
 *   expr := NAME | "(" ("AND"|"OR") operand+ ")" | "(" ("SOME"|"ONLY") ROLE expr ")"
 *         | "(" ("MIN"|"EXACTLY"|"MAX") INT ROLE expr ")"
 *         | "(" "DSOME" NUMROLE (">="|"=="|"<=") DECIMAL ")"
 *         | "(" "SSOME" STRROLE ("EQUAL"|"CONTAIN") STRING ")"
 *   operand := expr | "(" "NOT" NAME ")" ;  ROLE := NAME | "(" "INV" NAME ")"
 * extended with (NOT expr) for any expr (reading Q1), TOP, BOTTOM, empty
 * AND / OR, (DRANGE NUMROLE lo hi) (closed float32 interval, reading Q9; >=v, ==v, <=v
 * of DSOME are [v,+inf], [v,v], [-inf,v]) and nested (INV ROLE).  Numbers go through
 * strtof (reading Q8); STRING is "..." with backslash escaping the next byte.
 * `names` maps each kind of entity to its id (list index; NULL lists / NULL names =
 * the spelling c<id>, r<id>, d<id>, s<id>).  The hypotheses become roots 0..n_exprs-1
 * of one program, compiled as hedl_compile_ex (same flags).  Errors: HEDL_ERR_PARSE
 * (syntax, unknown name, negative or > 2^32-1 cardinality) with *err_index = the
 * hypothesis and *err_pos = the byte offset of the offending token (both only set on
 * PARSE / a null hypothesis); otherwise hedl_compile_ex's errors. */
typedef struct hedl_names {
    uint32_t n_concepts;
    const char *const *concepts;
    uint32_t n_roles;
    const char *const *roles;
    uint32_t n_data;
    const char *const *data;
    uint32_t n_strings;
    const char *const *strings;
} hedl_names;
hedl_status hedl_compile_text(const hedl_kb *kb, const hedl_names *names, const char *const *exprs, uint32_t n_exprs,
                              uint32_t flags, hedl_program **out, uint32_t *err_index, uint32_t *err_pos);

/* Device-side compile (the paper's future work: GPUs generate their own
 * evaluation plans).  Same program as hedl_compile, built on the KB's device from
 * DEVICE arrays (nodes / child_idx / roots as in hedl_compile, in device memory, read
 * on `stream`; the call synchronises `stream` before returning).  With
 * HEDL_COMPILE_HOST_INPUT the three arrays are HOST memory instead: the library
 * copies them to its scratch on `stream` (DMA straight from page-locked memory), so
 * host arrays -> program is one call (the e2e path of bench.py).  The input must list
 * children before parents (every child id < its parent's id: the post-order of
 * flattened trees), else BAD_EXPR.  String restrictions, AND/OR with > 64 operands
 * after flattening and inputs deeper than 512 levels are UNSUPPORTED (use
 * hedl_compile).  Other errors as hedl_compile (the lowest failing node is named).
 * The program is evaluated like any other; its plan is built on the device too. */
hedl_status hedl_compile_device(const hedl_kb *kb, const hedl_node *nodes, uint32_t n_nodes,
                                const uint32_t *child_idx, uint64_t n_child_idx,
                                const uint32_t *roots, uint32_t n_roots, uint32_t flags,
                                void *stream, hedl_program **out);

typedef struct hedl_program_info {
    uint32_t n_roots;
    uint32_t n_nodes;             /* computed canonical nodes after CSE */
    uint32_t n_levels;
    uint32_t n_bool, n_restrict, n_drange;
    double alg_bytes_total;       /* sum over roots of B(h) (per-hypothesis CSE only) */
    double alg_bytes_shared;      /* sum over canonical nodes (batch-wide CSE) */
    uint32_t n_string;            /* string restriction nodes (after EQUAL short-circuit) */
} hedl_program_info;
hedl_status hedl_program_get_info(const hedl_program *prog, hedl_program_info *out);
/* per-root algorithmic bytes B(h), host double[n] for roots [first, first+n) */
hedl_status hedl_program_root_bytes(const hedl_program *prog, uint32_t first, uint32_t n, double *out);

/* ---------------------------------------------------------------------------
 * Evaluation.  Counts per hypothesis: tp = |H & P|, fp = |H & N|,
 * fn = |P| - tp, tn = |N| - fp (Alg. 15).
 * ------------------------------------------------------------------------- */
typedef struct hedl_counts {
    uint64_t tp, fp, fn, tn;
} hedl_counts;

/* Latency path: evaluate one root.  out_bits: device u32[W] (nullable) receives
 * the instance bitset; out: HOST pointer, filled before return (the call
 * synchronises `stream`).  Errors: OUT_OF_RANGE (root), CUDA, OOM. */
hedl_status hedl_eval_one(const hedl_kb *kb, hedl_program *prog, uint32_t root,
                          uint32_t *out_bits, hedl_counts *out, void *stream);

/* eval_batch flags */
#define HEDL_EVAL_COUNTS_DEVICE 1u   /* `counts` is a device pointer; return after enqueue */
#define HEDL_EVAL_PER_NODE 2u        /* force the per-node kernels (disable lane-packed restrictions) */
#define HEDL_EVAL_FORCE_SLICE 4u     /* lane-pack every eligible restriction group, however small (tests) */
#define HEDL_EVAL_NO_FUSE 8u         /* materialise boolean fillers of lane packs instead of fusing them (A/B, tests) */
#define HEDL_EVAL_NO_RESTRICT_U 16u  /* restrictions never emit U rows: booleans over them run in full (A/B, tests) */
#define HEDL_EVAL_NO_USWEEP 32u      /* restrictions needed over one U set are swept over all rows (A/B, tests) */

/* Throughput path: evaluate roots [first_root, first_root + n_roots) of prog.
 * Output position i <-> root first_root + i (input order).
 * out_bits: device u32[n_roots][W] (nullable).  counts: host (default; the call
 * synchronises) or device (HEDL_EVAL_COUNTS_DEVICE; asynchronous) hedl_counts[n].
 * Results do not depend on chunking, CSE or flags. */
hedl_status hedl_eval_batch(const hedl_kb *kb, hedl_program *prog, uint32_t first_root,
                            uint32_t n_roots, uint32_t *out_bits, hedl_counts *counts,
                            void *stream, uint32_t flags);

/* Scores and top-k on the device (scoring for an on-GPU learner;
 * definitions are reading Q14 -- the paper itself reports covered examples only):
 *   HEDL_SCORE_ACCURACY  (tp + tn) / (tp + fp + fn + tn), 0 without examples
 *   HEDL_SCORE_F1        2 tp / (2 tp + fp + fn), 0 when the denominator is 0
 * in float64.  counts: DEVICE hedl_counts[n] (e.g. hedl_eval_batch with
 * HEDL_EVAL_COUNTS_DEVICE).  scores: DEVICE double[n] or NULL.  top_idx / top_scores:
 * DEVICE uint32[k] / double[k] (either may be NULL) = the k highest scores, descending,
 * ties broken by the lower index.  Requires k <= n and k <= 4096.  Asynchronous on
 * `stream` (device `device`).  Errors: INVALID_ARG, OOM, CUDA. */
#define HEDL_SCORE_ACCURACY 0u
#define HEDL_SCORE_F1 1u
hedl_status hedl_score_topk(const hedl_counts *counts, uint32_t n, uint32_t metric, uint32_t k, double *scores,
                            uint32_t *top_idx, double *top_scores, int device, void *stream);

/* ---------------------------------------------------------------------------
 * Device memory.  North_star: "PyTorch is used only for device memory, streams
 * and process groups" -- the library never owns a device allocator of its own
 * when the caller installs one.
 *
 * hedl_set_allocator: every device allocation of the library (KB arrays,
 * program workspaces, plans, device-compile scratch, score scratch) goes through
 * alloc(bytes, device, stream, ctx) -> device pointer (NULL = out of memory,
 * the call then fails with HEDL_ERR_OOM) and is released through
 * free(ptr, device, stream, ctx).  `device` is the CUDA device the block is for
 * (it is current during the call), `stream` the cudaStream_t of the API call
 * that needs it (blocks are used stream-ordered on that stream; a block is freed
 * only after the library's work on it is complete, or on the stream that used it
 * last).  Both NULL = the default, cudaMalloc / cudaFree.  The allocator can only
 * change while no KB is alive (else INVALID_ARG), so every block is freed by the
 * allocator that made it.  The Python binding installs torch's caching
 * allocator (torch.cuda.caching_allocator_alloc / _delete).
 * hedl_alloc_counters: device allocations / frees made so far (diagnostics and
 * the "no allocation after warm-up" tests). */
typedef void *(*hedl_dev_alloc_fn)(size_t bytes, int device, void *stream, void *ctx);
typedef void (*hedl_dev_free_fn)(void *ptr, int device, void *stream, void *ctx);
hedl_status hedl_set_allocator(hedl_dev_alloc_fn alloc, hedl_dev_free_fn free_fn, void *ctx);
hedl_status hedl_alloc_counters(uint64_t *n_alloc, uint64_t *n_free);

/* Caller-provided scratch (SURVEY 8(b) "Memory": latency calls never allocate).
 * hedl_program_workspace_bytes: device bytes one hedl_eval_batch(kb, prog, first_root,
 *   n_roots, ...) needs -- with_bits != 0 when out_bits will be requested, eval_flags
 *   the call's HEDL_EVAL_* flags (PER_NODE / FORCE_SLICE change the plan) -- computed
 *   by the planner's sizing pass, nothing launched.  hedl_eval_one needs the bytes of
 *   (root, 1, with_bits, HEDL_EVAL_PER_NODE) (its single-CTA path needs none).
 * hedl_program_set_workspace: `ptr` = DEVICE memory on the KB's device, `bytes` its
 *   size (>= 4 KiB), owned by the caller and kept alive until the program is freed or
 *   the workspace replaced (ptr NULL = back to library-allocated memory).  Every later
 *   evaluation of the program carves its buffers (rows, counts staging, lane-pack
 *   scratch, plan) out of this block and allocates no device memory; a call that needs
 *   more returns HEDL_ERR_OOM naming the size.  Calls on one program serialise, so one
 *   block serves any number of calls.  Both return HEDL_ERR_UNSUPPORTED for programs
 *   from hedl_compile_device (they plan on the device from the KB's pool). */
hedl_status hedl_program_workspace_bytes(const hedl_kb *kb, hedl_program *prog, uint32_t first_root,
                                         uint32_t n_roots, int with_bits, uint32_t eval_flags, uint64_t *bytes);
hedl_status hedl_program_set_workspace(hedl_program *prog, void *ptr, uint64_t bytes);

/* Device-memory cap for one program's evaluation workspace (default: half the
 * device memory free at first use, at most 48 GiB).  Larger caps give larger
 * chunks, i.e. fuller lane packs. */
hedl_status hedl_program_set_workspace_limit(hedl_program *prog, uint64_t bytes);

/* ---------------------------------------------------------------------------
 * Diagnostics
 * ------------------------------------------------------------------------- */
const char *hedl_last_error(void);
const char *hedl_version(void);

/* Kernel-level timing: when enabled, every kernel launch of the library is
 * bracketed by CUDA events on its launch stream; hedl_prof_read synchronises
 * and returns per kernel class {name, launches, total_ms, alg_bytes, units}. */
typedef struct hedl_prof_entry {
    char name[32];
    uint64_t launches;
    double total_ms;
    double alg_bytes;
    double units;          /* work units launched: nodes for per-node kernels and packs; for the lane-packed
                              sweeps (slice, slice_heavy, slice_ex, slice_u) the bytes of T gathered,
                              32 B per swept edge and pack (the L2-gather traffic of the sweep) */
} hedl_prof_entry;
hedl_status hedl_prof_enable(int on);
hedl_status hedl_prof_reset(void);
int hedl_prof_read(hedl_prof_entry *out, int max_entries);
/* number of library kernel launches since process start (always counted) */
uint64_t hedl_launch_count(void);
/* bytes the library copied host->device / device->host since process start */
hedl_status hedl_io_counters(uint64_t *h2d_bytes, uint64_t *d2h_bytes);

#ifdef __cplusplus
}
#endif
#endif /* HEDL_H */

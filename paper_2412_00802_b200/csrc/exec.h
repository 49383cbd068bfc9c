// Executor internals shared by the host planner (exec.cu) and the device planner (dplan.cu).
#pragma once
#include "internal.h"

namespace hedl {

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

struct LaunchRec {
    uint8_t kind;          // NK_AND (AND+OR), NK_RESTRICT, NK_DRANGE, NK_STRING
    uint16_t key;          // dir / prop
    bool slice;
    bool proj;             // boolean group evaluated on example-projected rows
    bool ex;               // restriction pack evaluated on example rows only
    uint32_t count, first_desc;
    double bytes, bytes2;
    int8_t cls = -1;       // lane-pack class of the whole group (device plans), -1 = per descriptor
    int16_t usp = -1;      // boolean group over U of direction usp
    bool ucomp = false;    // EX pack reading its fillers' U rows
    int8_t usw = -1;       // U-sweep pack (rows of U_usw only)
};

struct ChunkPlan {
    uint32_t ri, rc;       // roots [ri, rc) relative to the program
    uint32_t nn, ncov, nrows, nprows;
    size_t blob_off, blob_bytes;          // into PlanCache host/device blobs
    size_t off_bool, off_ops, off_res, off_dr, off_str, off_cov, off_rows;
    uint32_t nurows = 0, nurows_r = 0;   // U rows; the first nurows_r are restrictions' (zeroed per chunk)
    std::vector<LaunchRec> recs;
};

struct PlanCache {
    bool valid = false;
    uint32_t r0 = 0, r1 = 0, eflags = 0;
    bool bits = false;
    void *rows_base = nullptr, *heavy_base = nullptr, *prows_base = nullptr, *urows_base = nullptr;
    std::vector<ChunkPlan> chunks;
    void *host = nullptr;                 // pinned descriptor blob
    void *dev = nullptr;                  // device descriptor blob
    size_t cap = 0;                       // capacity of both blobs
    size_t host_cap = 0;                  // capacity of the host blob (caller-workspace mode)
    // the plan's launches captured as a CUDA graph (replayed by later calls with the same
    // output buffers): one graph launch instead of ~250 kernel launches per C4 step
    cudaGraphExec_t graph = nullptr;
    const void *g_counts = nullptr, *g_bits = nullptr;
    uint32_t g_calls = 0;                 // replays seen: capture from the second one on
    uint64_t g_launches = 0;              // kernels in the graph (the launch counter's share)
    // the graph runs on the library's own stream, ordered after / before the caller's stream by
    // events (the legacy default stream a caller usually passes cannot be captured)
    cudaStream_t gstream = nullptr;
    cudaEvent_t gev_in = nullptr, gev_out = nullptr;
};

struct Workspace {
    DevBuf rows, prows, heavy, counts, slice, stage, urows;
    uint8_t *pats = nullptr;             // device copy of the program's CONTAIN patterns
    std::vector<uint64_t> pat_off;       // their offsets
    hedl_counts *stage_host = nullptr;   // pinned staging of host-bound counts
    size_t stage_host_n = 0;
    PlanCache plan;
    cudaEvent_t done = nullptr;
    cudaStream_t last_stream = nullptr;
    bool used = false;
    // caller-provided device block (hedl_program_set_workspace): while set, every buffer
    // above (and the device plan blob, the pattern table) is carved out of it, re-carved
    // from its start whenever the plan is rebuilt; nothing is allocated or freed
    char *ext = nullptr;
    size_t ext_bytes = 0, ext_used = 0;
};

Workspace *ws_of(hedl_program *p);
hedl_status grow(const hedl_kb *kb, cudaStream_t s, DevBuf &b, size_t need, bool zero, int role, Workspace *w = nullptr);
void invalidate_plan(PlanCache &pc);
void release_plan(PlanCache &pc);
hedl_status reserve_plan(const hedl_kb *kb, PlanCache &pc, size_t bytes, Workspace *w = nullptr);
hedl_status launch_chunk(const hedl_kb *kb, Workspace *w, const ChunkPlan &cp, uint32_t r0, uint32_t *out_bits,
                         hedl_counts *counts_dev, cudaStream_t s);
// the launches of a valid plan: its captured graph when possible, else launch_chunk per chunk
hedl_status replay_plan(const hedl_kb *kb, Workspace *w, uint32_t r0, uint32_t *out_bits, hedl_counts *counts_dev,
                        cudaStream_t s);
void drop_graph(PlanCache &pc);
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
// scratch of a per-node restriction group of `count` nodes in direction `dir`: the heavy-row
// counters, then (small groups on large KBs) the push-direction scratch of each node
inline bool restrict_push(const hedl_kb *kb, uint32_t count) { return count <= kPushMaxNodes && kb->N >= kPushMinN; }
inline size_t restrict_heavy_bytes(const hedl_kb *kb, uint32_t dir, uint32_t count) {
    return align_up((size_t)count * kb->dirs[dir].n_heavy * 8, 256);
}
inline size_t restrict_scratch_bytes(const hedl_kb *kb, uint32_t dir, uint32_t count) {
    size_t b = restrict_heavy_bytes(kb, dir, count);
    if (restrict_push(kb, count)) b += (size_t)count * push_scratch_words(kb->N, kb->W4, true) * 4;
    return b;
}
// device planner (dplan.cu): builds and launches the plan of a device-compiled program on
// the device; HEDL_ERR_UNSUPPORTED = the batch does not fit one chunk (host planner then)
hedl_status dplan_run(const hedl_kb *kb, hedl_program *p, uint32_t r0, uint32_t r1, uint32_t *out_bits,
                      hedl_counts *counts_dev, cudaStream_t s, uint32_t eflags);
void dplan_free(hedl_program *p);

}  // namespace hedl

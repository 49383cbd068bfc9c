// Latency-path interpreter (interp.cu): a root's sub-DAG as a kernel parameter.
#pragma once
#include "internal.h"

namespace hedl {
constexpr uint32_t kInterpMaxNodes = 96, kInterpMaxOps = 512;
constexpr uint32_t kInterpMaxN = 1u << 16;   // individuals; larger KBs use the per-node kernels
constexpr uint32_t kInterpCl = 8;            // CTAs of the cluster interpreter
constexpr uint32_t kInterpClusterMinW4 = 256;   // rows of at least this many words use it

struct InterpNode {
    uint8_t kind, pred;     // kind bit 7: a restriction reads this row at any individual
    uint16_t dir;
    uint32_t n, sat;
    float lo, hi;
    uint32_t op_begin, op_count;   // operand refs: RT_NODE ids are local (topological) indices
};

struct InterpProg {
    uint32_t n_nodes, n_ops;
    uint64_t npos, nneg;
    uint64_t seq;              // written to counts[1].tp (mapped host memory) after the counts
    InterpNode nodes[kInterpMaxNodes];
    uint32_t ops[kInterpMaxOps];
};

size_t interp_smem_limit();
hedl_status interp_prepare(hedl_kb *kb);
hedl_status interp_launch(const hedl_kb *kb, const InterpProg &prog, hedl_counts *counts_mapped, uint32_t *out_bits,
                          cudaStream_t s);
}  // namespace hedl

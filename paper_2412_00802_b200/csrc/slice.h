// Lane-packed ("bit-sliced") batch restriction path (SURVEY 8(d) "Optional
// bit-sliced batch variant"): many restriction nodes on one role direction
// share one CSR pass.  Declarations; implementation in slice.cu.
#pragma once
#include "internal.h"

namespace hedl {
constexpr uint32_t kSliceMinNodes = 8;   // smaller groups use the per-node kernels
bool slice_enabled(const hedl_kb *kb);
bool slice_worthwhile(const hedl_kb *kb, uint32_t n_nodes, bool force);
// 0 = OR pack (count saturates at 1), 1 = COUNT pack (n <= 30), 2 = per-node kernel
uint32_t slice_class(uint32_t pred, uint32_t n, uint32_t sat);
// h_desc: host copies of the group's restriction descriptors (pinned, valid
// until the stream reaches this point); d_desc: the same on the device.
// fixed_cls >= 0: every descriptor has this class (h_desc may be null).
// ucomp (EX packs): the descriptors' child rows are U rows of this direction (DESIGN.md
// "U-projected rows"), else full rows compacted to U while packing.
// d_ops: the plan's operand table, read for fused fillers (descriptors with child == null).
// usw >= 0: a U-sweep group (full T; rows of U_usw only; results to the nodes' U rows in proj).
// bytes of the lane-pack scratch (T, heavy accumulators, scheduler) a KB's packs need
size_t slice_ws_bytes(const hedl_kb *kb);
hedl_status slice_run(const hedl_kb *kb, void **ws, size_t *ws_bytes, cudaStream_t s, const KbDev &kd,
                      uint32_t dir, const RestrictDesc *h_desc, const RestrictDesc *d_desc, uint32_t n,
                      hedl_counts *counts, bool ex, int fixed_cls = -1, bool ucomp = false,
                      const Operand *d_ops = nullptr, int usw = -1);
}  // namespace hedl

// Lane-packed batch restriction kernels (placeholder until implemented).
#include "slice.h"

namespace hedl {
bool slice_enabled(const hedl_kb *) { return false; }
bool slice_worthwhile(const hedl_kb *, uint32_t) { return false; }
hedl_status slice_run(const hedl_kb *, void **, size_t *, cudaStream_t, const KbDev &, uint32_t,
                      const RestrictDesc *, const RestrictDesc *, uint32_t, hedl_counts *) {
    return fail(HEDL_ERR_UNSUPPORTED, "lane-packed path not built");
}
}  // namespace hedl

// nvtx.cuh -- NVTX ranges per stage and per gadget call (stage
// timing under nsys / ncu --nvtx). Header-only NVTX v3: without an attached
// tool a range costs one indirect call.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace sz {
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace sz
#define SZ_RANGE_CAT2(a, b) a##b
#define SZ_RANGE_CAT(a, b) SZ_RANGE_CAT2(a, b)
#define SZ_RANGE(name) ::sz::NvtxRange SZ_RANGE_CAT(sz_nvtx_, __LINE__)(name)

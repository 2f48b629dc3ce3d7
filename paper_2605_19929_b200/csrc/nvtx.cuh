// NVTX ranges around the host-side launch sequence (K1, LR1, split GEMM,
// MOCD statistics), so an Nsight timeline names each stage. NVTX v3 is
// header-only: without an attached tool the calls are no-ops.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace splitq {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
  // end this range and open the next stage's (one range open at a time)
  void next(const char* name) {
    nvtxRangePop();
    nvtxRangePushA(name);
  }
};
}  // namespace splitq

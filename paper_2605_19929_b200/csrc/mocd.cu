// MOCD calibration statistics (placeholder until the K6 kernels land).
#include "../../include/splitq.h"
extern "C" {
int splitq_mocd_absmax(const void*, int, int64_t, const uint8_t*, int64_t, int64_t, float*, float*,
                       int32_t*, void*) { return SPLITQ_ERR_UNSUPPORTED; }
int splitq_mocd_rank_counts(const void*, int, int64_t, const int32_t*, const int32_t*, int64_t,
                            const int32_t*, int64_t, uint16_t*, void*) { return SPLITQ_ERR_UNSUPPORTED; }
int splitq_mocd_histogram(const uint16_t*, const int32_t*, int64_t, int64_t, int32_t*, void*) {
  return SPLITQ_ERR_UNSUPPORTED;
}
int splitq_mocd_text_score(const int32_t*, int64_t, int64_t, int, int, double*, void*) {
  return SPLITQ_ERR_UNSUPPORTED;
}
}

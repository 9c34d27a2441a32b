// Internal definition of the opaque mg_mt64 handle (include/mgcuda.h).
#pragma once

#include <stdint.h>

#include "mgcuda.h"

struct mg_mt64 {
  int32_t streams = 0;
  uint64_t* state = nullptr;  // device [streams][312]
  int* idx = nullptr;         // device [streams]
  int host_idx = 312;         // common position of all streams in their block (1..312)
};

namespace mg {
int mt64_create(mg_ctx* ctx, int32_t streams, const uint64_t* host_seeds, mg_mt64** out);
void mt64_destroy(mg_mt64* g);
int mt64_draw(mg_ctx* ctx, mg_mt64* g, int64_t n, int32_t kind, void* out);
int mt64_jump(mg_ctx* ctx, mg_mt64* g, uint64_t distance, const uint8_t* dev_mask);
}  // namespace mg

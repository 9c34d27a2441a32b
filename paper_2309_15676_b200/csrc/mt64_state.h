// Internal definition of the opaque mg_mt64 handle (include/mgcuda.h).
#pragma once

#include <stdint.h>

#include "mgcuda.h"

struct mg_mt64 {
  int32_t streams = 0;
  uint64_t* state = nullptr;  // device [streams][312]
  int* idx = nullptr;         // device [streams]
};

namespace mg {
int mt64_create(mg_ctx* ctx, int32_t streams, const uint64_t* host_seeds, mg_mt64** out);
void mt64_destroy(mg_mt64* g);
int mt64_draw(mg_ctx* ctx, mg_mt64* g, int64_t n, int32_t kind, void* out);
}  // namespace mg

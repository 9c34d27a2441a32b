// Shared between the fused mini-render kernels (render.cu: IEEE, every
// dtype / RNG mode; render_fast.cu: the fp32 Philox TMA-fed kernel).
#pragma once

#include <stdint.h>

#include "meta_math.cuh"
#include "mg_common.cuh"

namespace mg {

struct RenderK {
  MetaK meta;
  int spp;
  int philox;  // 0: uniforms buffer (mt19937_64 stream), 1: Philox counter
  uint64_t key;
  uint32_t iteration, stream, pixel_offset;
  int64_t record;  // -1: full prop/diff outputs, else only this local pixel
};

extern bool g_render_fast;
extern int g_render_fast_variant;

// fp32, no per-pixel outputs (Philox draws, or the mt64 draws streamed).  Returns MG_EUNSUPPORTED when
// the launch does not fit the fast kernel (spp > 4, unaligned views, P below
// one tile per SM); the caller then runs the IEEE kernel.
// uniforms: the pre-drawn mt19937_64 draws (mt64 mode, pixel-major, 16-byte
// aligned), ignored in Philox mode.
int launch_minirender_fast(mg_ctx* ctx, int64_t P, const RenderK& k, bool first, const float* b,
                           const float* tgt, const float* pnow, float* pprev_next, float* m2p,
                           float* m2d, float* mean, float* var, float* ap, mg_update_scalars* sc,
                           const double* uniforms);

}  // namespace mg

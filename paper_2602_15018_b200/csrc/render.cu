// GPU ray caster for the frame producer: the
// reference's render_pair (/root/reference/pkg/src/evsim/render.py:179-208)
// -- axis-aligned textured planes (checkerboard, value noise), pinhole
// camera, projective z-depth -- so frames are born in HBM next to the event
// path instead of crossing PCIe.  f64 arithmetic in the reference's operation
// order with explicit roundings (no FMA contraction); the only expected
// difference is the ray direction's 3-term dot product, which numpy evaluates
// through BLAS (render.py:176).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../../include/evsim_b200.h"

namespace {

__device__ __forceinline__ double hash01(int64_t ix, int64_t iy, uint64_t seed_mix) {
  // render.py:111-120 (_hash01)
  uint64_t h = ((uint64_t)ix * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)iy * 0xC2B2AE3D27D4EB4Full) ^ seed_mix;
  h ^= h >> 33;
  h *= 0xFF51AFD7ED558CCDull;
  h ^= h >> 33;
  return __ddiv_rn((double)(h >> 11), 9007199254740992.0);  // / 2^53
}

__device__ __forceinline__ double tex_sample(const evs_plane& pl, double a, double b) {
  if (pl.kind == EVS_TEX_CHECKER) {  // render.py:72-74
    const int64_t par = ((int64_t)floor(__ddiv_rn(a, pl.cell)) + (int64_t)floor(__ddiv_rn(b, pl.cell))) & 1;
    return par == 0 ? pl.value_a : pl.value_b;
  }
  // render.py:92-108 (ValueNoise.sample)
  const double qa = __ddiv_rn(a, pl.cell), qb = __ddiv_rn(b, pl.cell);
  const double fia = floor(qa), fib = floor(qb);
  const double fa = __dsub_rn(qa, fia), fb = __dsub_rn(qb, fib);
  const int64_t ia = (int64_t)fia, ib = (int64_t)fib;
  const uint64_t sm = pl.seed * 0xD6E8FEB86659FD93ull;
  const double v00 = hash01(ia, ib, sm), v10 = hash01(ia + 1, ib, sm);
  const double v01 = hash01(ia, ib + 1, sm), v11 = hash01(ia + 1, ib + 1, sm);
  const double top = __dadd_rn(v00, __dmul_rn(__dsub_rn(v10, v00), fa));
  const double bot = __dadd_rn(v01, __dmul_rn(__dsub_rn(v11, v01), fa));
  const double val = __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), fb));
  return __dadd_rn(pl.value_a, __dmul_rn(__dsub_rn(pl.value_b, pl.value_a), val));  // lo + (hi - lo) * val
}

__global__ void __launch_bounds__(256) k_render(evs_render_params p, const evs_plane* __restrict__ planes,
                                               int nplanes, float* __restrict__ intensity,
                                               float* __restrict__ depth) {
  const int64_t n = (int64_t)p.width * p.height;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx / p.width), i = (int)(idx - (int64_t)j * p.width);
    // render.py:166-176: camera ray with z = 1, rotated to the world frame
    const double u = __ddiv_rn(__dsub_rn((double)i, p.cx), p.fx);
    const double v = __ddiv_rn(__dsub_rn((double)j, p.cy), p.fy);
    double d[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
      d[r] = __dadd_rn(__dadd_rn(__dmul_rn(u, p.rot[3 * r + 0]), __dmul_rn(v, p.rot[3 * r + 1])), p.rot[3 * r + 2]);
    double best = INFINITY;
    double inten = p.ambient;
    for (int q = 0; q < nplanes; ++q) {  // render.py:185-203, declaration order (ties keep the first)
      const evs_plane pl = planes[q];
      const int k = pl.axis;
      const int a1 = k == 0 ? 1 : 0, a2 = k == 2 ? 1 : 2;
      const double dk = d[k];
      const double tt = __ddiv_rn(__dsub_rn(pl.offset, p.origin[k]), dk);
      const double pa = __dadd_rn(p.origin[a1], __dmul_rn(tt, d[a1]));
      const double pb = __dadd_rn(p.origin[a2], __dmul_rn(tt, d[a2]));
      const bool hit = isfinite(tt) && tt > 1e-9 && tt < best && pa >= pl.bounds[0] && pa <= pl.bounds[1] &&
                       pb >= pl.bounds[2] && pb <= pl.bounds[3];
      if (hit) {
        best = tt;
        inten = tex_sample(pl, pa, pb);
      }
    }
    inten = fmin(fmax(inten, 0.0), 1.0);  // render.py:204
    intensity[idx] = (float)inten;
    if (depth) depth[idx] = (float)best;
  }
}

}  // namespace

extern "C" evs_status evs_render(const evs_render_params* p, const evs_plane* planes, int32_t nplanes,
                                 float* intensity, float* depth, void* stream) {
  if (!p || !intensity || p->width < 1 || p->height < 1 || nplanes < 0 || (nplanes > 0 && !planes))
    return EVS_ERR_ARG;
  const int64_t n = (int64_t)p->width * p->height;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_render<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(*p, planes, nplanes, intensity, depth);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

// Fast canonical-order path (fast_path.cu): constants, argument block, launchers.
//
// Error model of the certified f32 lane math (K1):
//   x = f64(v) + log_eps is formed exactly as the reference does; ln(x) is
//   k*ln2 + log(c_i) (f64) + log1p(r) with r = (x/2^k - c_i)/c_i, |r| <= 2^-7,
//   evaluated in f32 (degree 5, truncation < 4e-14, rounding < 2^-30).  With the
//   reference's own log within 2 ulp, |df - diff_ref| <= 4e-9 + 2*2^-24*|df|.
//   K1 uses kEpsD = 8e-9 and relative slack 8*2^-24 (the reciprocal is
//   rcp.approx, <= 1 ulp) for the bands of n = floor(|d|/th + 1e-4) and of
//   t_rel = floor(j*th*dt/|d|); a straddling band sends the pixel to the exact
//   path (f64 log <= 1 ulp, IEEE division, the reference's operation order).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace evs {

constexpr int kFNT = 256;                 // K1 threads per CTA
constexpr int kFVpt = 4;                  // pixels per thread (one float4)
constexpr int kFCtasPerSm = 3;            // K1 residency target (smem, 64 registers)
constexpr int kFGmax = kFNT * kFVpt;      // max pixels per tile (2048; local index fits 11 bits)
constexpr int kFListCap = 5 * kFGmax;     // crossings per tile-frame held in smem (kFListCap/16 per warp)
constexpr bool kFPrefilter = false;       // f32 __logf prefilter before the lite math
constexpr int kFMaxBuckets = 256;         // buckets of 8 t_rel bins: dt <= 2048 us
constexpr int kFMaxTiles = 4096;          // tiles per stream (K2 smem tables)
constexpr int kONT = 512;                 // K2 threads per CTA
constexpr int kOCap = 12288;              // K2 entries per chunk (smem)

constexpr int64_t kSrcSlot = -1, kSrcRedo = -3;

// sorted-key layout (4 bytes): t_rel << 12 | local pixel << 1 | (p > 0); bucket = key >> 15

struct FastArgs {
  int S, T, W, G, ntiles, nbk, vec;
  int64_t P;
  double log_eps;
  float log_eps_f;
  int refr;
  float thp_u, thn_u, rthp_u, rthn_u;
  const float* frames;       // [S][T][P]
  const int64_t* t_bounds;   // [S][T+1] or null
  int64_t t0, tick;
  const StepDesc* desc;      // device clock or null
  float* ref;                // [S][P] in/out
  int64_t* last;             // [S][P] in/out
  const float* thp;          // [S][P] or null (uniform)
  const float* thn;
  const int64_t* bad;        // first invalid pixel (prologue)
  int64_t* seg_res;          // [nseg] reservation chunks
  uint32_t* keys;            // [nseg][ntiles][kFListCap] bucket-sorted keys
  uint32_t* rows;            // [nseg][nbk+1][ntiles] bucket starts per tile (row nbk = tile total)
  int64_t* tile_src;         // [nseg][ntiles] kSrcSlot: keys slot; kSrcRedo: regenerate; >= 0: area offset
  // tile-frames whose crossings exceed kFListCap: K1 leaves the state before
  // the frame, k_fast_redo regenerates the kept share into the area
  float* snap_ref;           // [nseg][ntiles][G]
  int* snap_last;            // [nseg][ntiles][G] (relative to the call's first t_prev)
  uint32_t* area_unsorted;   // [nseg][cap]
  uint32_t* area_sorted;     // [nseg][cap]
  int* redo_items;           // [nseg][ntiles][2] (tile, area offset)
  int* redo_lim;             // [nseg][ntiles] kept share of each redo tile
  int* redo_n;               // [nseg]
  uint32_t* btot;            // [nseg][nbk] events per bucket (zeroed by the prologue)
  // K2 work split: pieces of <= ~kOCap events (a bucket, or a tile range of a big bucket)
  int* pieces;               // [nseg][maxp][8]: k, qa, qb, j0, j1, big
  int* npieces;              // [nseg]
  uint32_t* pcnt;            // [nseg][maxp][8] per-bin counts of big-bucket pieces
  int maxp;
  int64_t cap;               // events kept per segment
  int64_t* out_count;
  int64_t* out_dropped;
  int64_t seg_stride;
  int64_t* out_t;
  uint16_t* out_x;
  uint16_t* out_y;
  int8_t* out_p;
};

size_t fast_gen_smem();
size_t fast_order_smem(int ntiles);
cudaError_t launch_fast_gen(const FastArgs& a, cudaStream_t st);
cudaError_t launch_fast_fix(const FastArgs& a, int nseg, cudaStream_t st);
cudaError_t launch_fast_redo(const FastArgs& a, int nseg, cudaStream_t st);
cudaError_t launch_fast_plan(const FastArgs& a, int nseg, cudaStream_t st);
cudaError_t launch_fast_order(const FastArgs& a, int nseg, cudaStream_t st);

}  // namespace evs

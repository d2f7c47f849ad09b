// Kernel argument blocks and launch helpers shared by the .cu files.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace evs {

constexpr int64_t kNoBad = 0x7fffffffffffffffLL;
constexpr int kHistReps = 8;      // replicated global histograms (atomic spread)
// crossings of one pixel in one frame: <= (ln(1 + eps) - ln(eps)) / 0.01 + 1 for
// a reference level inside the log range (462 at eps = 0.01, MIN_THRESHOLD);
// more only comes from a corrupt level and fails the call (no 32-bit overflow)
constexpr int64_t kMaxPixelCrossings = 1 << 20;
constexpr int kMaxDigitBits = 11; // onesweep digit width (<= 2048 bins)
constexpr int kKeyPixBits = 33;   // key = t_rel << 33 | y << 17 | x << 1 | (p > 0)

constexpr int kGenThreads = 256;
constexpr int kGenVpt = 4;
constexpr int kGenTile = kGenThreads * kGenVpt;  // pixels per K1 tile (the largest; small sensors use
                                                 // 256-pixel tiles, one pixel per thread: args.tile_px)

constexpr int kOrdThreads = 256;
constexpr int kOrdIpt = 16;
constexpr int kOrdTile = kOrdThreads * kOrdIpt;  // keys per K2 tile

// Raise a kernel's dynamic shared-memory limit to the opt-in maximum, once per
// (device, kernel); thread-safe (k1_list.cu).
void smem_optin(const void* func);

// Device-resident step clock (EVS_FLAG_DEVICE_CLOCK): lets a captured CUDA
// graph replay steps whose start time and lookback epoch advance on device.
struct StepDesc {
  int64_t next_t0, cur_t0;
  uint32_t next_epoch, cur_epoch;
};

struct GenArgs {
  int tile_px, tile_cap;  // pixels per K1 tile (1024 or 256) and keys per tile region (4 per pixel)
  int S, T, H, W;
  int64_t P;
  double log_eps;
  int64_t refr, cap;
  float thp_u, thn_u;
  const float* frames;      // [S][T][P]
  const int64_t* t_bounds;  // [S][T+1] or null
  int64_t t0, tick;
  float* ref;
  int64_t* last;
  const float* thp;
  const float* thn;
  int mode;  // 0: SoA pixel-major, 1: keys to scratch
  int64_t* out_t;
  uint16_t* out_x;
  uint16_t* out_y;
  int8_t* out_p;
  uint64_t* keys;
  int64_t seg_stride;
  int64_t* seg_total;  // [S*T] kept events before capacity
  int64_t* seg_res;    // [S*T] reservation chunks
  int64_t* seg_tbase;  // [S*T] t_prev of each segment
  uint32_t* hist;      // [S*T][npass][R][NB] (pass 0) or null
  int npass, hist_bits;
  uint64_t* status;  // [S*T][ntiles]
  uint32_t* tile_ctr;
  const int64_t* bad;
  uint32_t epoch;
  int ntiles;  // tiles per stream frame
  const StepDesc* desc;  // non-null: t0 / epoch come from the device clock
  // per tile-group t_rel histogram rows (canonical order, pass 0):
  // rows[seg][group][NB], group = tile / gt -- filled by k_group_hist, carried
  // here for the later passes' arguments (K1 itself does not touch them)
  uint32_t* rows;
  int64_t* group_base;
  int ngroups;
  float log_eps_f;  // log_eps rounded to f32 (prefilter only)
  double rth_pos, rth_neg;  // 1/th for uniform thresholds (set by launch_generate)
  float rthp_f, rthn_f;     // the same rounded to f32 (certified lite math)
  double w_inv;             // 1 / W (set by launch_generate)
  float thp_pf, thn_pf;     // th * (1 - 1e-4) of the uniform thresholds (prefilter)
  int64_t max_dt;           // bound of t_now - t_prev over the call (params.max_dt, else tick)
  // per-tile event regions (no inter-tile dependency in K1):
  uint64_t* region;          // [nseg][ntiles][kTileCap] pixel-major keys
  int64_t* tile_count;       // [nseg][ntiles] events of the tile (before capacity)
  int64_t* tile_ovf;         // [nseg][ntiles] -1, or offset into ovf_area (lane slot overflow)
  uint64_t* ovf_area;        // [nseg][ovf_cap] spill: K1 claims [0, ovf_lim), regenerated tiles follow
  unsigned long long* ovf_cursor;  // [nseg], zeroed by the prologue
  int64_t ovf_cap, ovf_lim;
  int64_t* err;              // [1] bit 1: corrupt level (> kMaxPixelCrossings)
  unsigned int* ticket;      // CTA ticket (zeroed by the prologue): work in dispatch order
  int64_t* seg_dt;           // [S*T] t_now - t_prev of each segment
  // tiles that found the spill area full: pre-frame state for their regeneration
  float* snap_ref;           // [nseg][ntiles][kGenTile]
  int32_t* snap_last;        // [nseg][ntiles][kGenTile] last event - t_prev, clamped to [-2^30, 2^30]
  int gt;                    // tiles per group (histogram row)
  // frame chunking: block b handles chunk c = b / (S*ntiles) = frames
  // [c*tc, min(T, (c+1)*tc)) of its tile; chunk c waits for chunk c-1 of the
  // same tile through chunk_flag[(s, tile)] = (launch << 8) | chunks_done
  int nchunks, tc;
  unsigned long long* chunk_flag;  // [S*ntiles]
  // fused validation (model.py:28-39 semantics without a separate pass over the
  // frames): K1 checks every value it loads (atomicMin of the first bad flat
  // index), frame chunk 0 saves the call's initial state here, and k_tilescan
  // restores it when some value was invalid (the state is then untouched).
  int fuse_validate;
  int64_t* bad_rw;
  float* bak_ref;      // [S][P]
  int64_t* bak_last;   // [S][P]
};

constexpr int64_t kTileRedo = -3;  // tile_ovf: K1 kept only the count (k_group_hist regenerates)
constexpr int kTileCap = 4 * kGenTile;  // keys per region of the largest tile (4 per pixel; args.tile_cap)

struct TileScanArgs {
  int tile_px, tile_cap;  // pixels per K1 tile (1024 or 256) and keys per tile region (4 per pixel)
  int nseg, ntiles, ngroups, bits;
  int64_t cap;
  const int64_t* tile_count;  // [nseg][ntiles]
  const int64_t* tile_ovf;
  const uint64_t* region;
  const uint64_t* ovf_area;
  int64_t ovf_cap;
  int64_t* tile_base;         // out [nseg][ntiles] pixel-major base of each tile
  uint32_t* rows;             // [nseg][ngroups][NB] (null: counts only)
  uint32_t* tot;              // out [nseg][NB]
  int64_t* out_count;
  int64_t* out_dropped;
  const int64_t* bad;
  const int64_t* err;         // K1 errors -> out_dropped = -2 (corrupt level)
  int gt;                     // tiles per group (histogram row, K2 CTA)
  int rows_stride;            // groups per segment in the rows array (>= ngroups)
  // regeneration of tiles K1 could not store (tile_ovf == kTileRedo, or
  // >= ovf_lim once regenerated): k_group_hist, when ovf_cursor[seg] > ovf_lim
  int64_t ovf_lim;
  const unsigned long long* ovf_cursor;
  int64_t* err_rw;
  const float* frames;
  int T, W;
  int64_t P;
  const float* thp;
  const float* thn;
  float thp_u, thn_u;
  double log_eps;
  int refr;
  const int64_t* seg_tbase;
  const int64_t* seg_dt;
  const float* snap_ref;
  const int32_t* snap_last;
  // fused validation: restore the state from the backup when a frame was invalid
  const float* bak_ref;
  const int64_t* bak_last;
  float* ref;
  int64_t* last;
  int64_t sp;                 // S * P (0: no restore)
};

struct TileOrderArgs {
  int tile_px, tile_cap;  // pixels per K1 tile (1024 or 256) and keys per tile region (4 per pixel)
  int nseg, ntiles, ngroups, bits, shift;
  int64_t cap;
  const int64_t* tile_count;
  const int64_t* tile_ovf;
  const int64_t* tile_base;
  const uint64_t* region;
  const uint64_t* ovf_area;
  int64_t ovf_cap;
  uint32_t* rows;
  const uint32_t* tot;
  int64_t seg_stride;         // output stride per segment
  int final_soa;              // 1: SoA out; 0: keys_out
  int pixel_major;            // 1: plain compaction (serial order), no t ordering
  uint64_t* keys_out;
  int64_t* out_t;
  uint16_t* out_x;
  uint16_t* out_y;
  int8_t* out_p;
  const int64_t* seg_tbase;
  const int64_t* bad;
  int gt;
  int rows_stride;            // as TileScanArgs
};

// Voxel grid of one stream's window straight from a step's per-tile key
// regions (represent.cu): one CTA per 1024-pixel tile accumulates the exact
// int64 numerators of its own pixels in shared memory (no global atomics).
struct StepVoxArgs {
  int tile_px, tile_cap;  // pixels per K1 tile (1024 or 256) and keys per tile region (4 per pixel)
  int ntiles, T, s, B;
  int W;
  int64_t P, cap, ovf_cap;
  const int64_t* tile_count;
  const int64_t* tile_base;
  const int64_t* tile_ovf;
  const uint64_t* region;
  const uint64_t* ovf_area;
  const int64_t* seg_tbase;
  const int64_t* bad;
  int64_t t0, t1;
  long long* acc_out;  // [B][P] int64 numerators (stored), or null
  float* out;          // [B][P] f32 result, or null
};
constexpr int kStepVoxMaxBins = 24;
cudaError_t launch_step_voxel(const StepVoxArgs& a, cudaStream_t st);
cudaError_t launch_step_hist(const StepVoxArgs& a, int S, int64_t lo, int64_t hi, int64_t* out, cudaStream_t st);
cudaError_t launch_group_hist(const TileScanArgs& a, cudaStream_t st);
cudaError_t launch_tilescan(const TileScanArgs& a, cudaStream_t st);
int tile_order_chunk_keys(int tile_px, int pixel_major, int bits);  // keys per K2 chunk of that launch
cudaError_t launch_tile_order(const TileOrderArgs& a, cudaStream_t st);

constexpr int kMaxGroupTiles = 16;  // K1 tiles per histogram row / per K2 CTA (runtime gt <= this)

struct PlanArgs {
  int nseg;
  int64_t cap;
  const int64_t* seg_total;
  int64_t* out_count;
  int64_t* out_dropped;
  const uint32_t* hist;  // [nseg][npass][R][NB] or null
  int npass, pass, bits;
  uint32_t* gstart;           // [nseg][NB]
  uint32_t* seg_tile_prefix;  // [nseg+1]
  const int64_t* bad;
  int zero_hist;
};

struct OrderArgs {
  int nseg;
  const uint64_t* keys_in;
  int64_t seg_stride;
  const int64_t* seg_count;
  const uint32_t* seg_tile_prefix;
  const uint32_t* gstart;
  int shift, bits;
  uint64_t* status;  // [nseg][max_tiles][NB]
  int64_t max_tiles;
  uint32_t* ctr;
  uint32_t epoch;
  int final_soa;
  uint64_t* keys_out;
  int64_t* out_t;
  uint16_t* out_x;
  uint16_t* out_y;
  int8_t* out_p;
  const int64_t* seg_tbase;
  const StepDesc* desc;  // non-null: epoch = desc->cur_epoch + epoch
};

struct HistArgs {
  int nseg;
  const uint64_t* keys;
  int64_t seg_stride;
  const int64_t* seg_count;
  int npass, pass0, bits;  // histogram passes [pass0, npass)
  int base_shift;          // bit position of pass 0's digit
  uint32_t* hist;          // [nseg][npass][R][NB]
};

// host launchers (k1_list.cu, order.cu)
cudaError_t launch_prologue(const float* frames, int64_t nframes, int64_t P, int validate,
                            int64_t* bad, int64_t* seg_res, int nseg, StepDesc* desc,
                            int64_t t_advance, int64_t* zero2, int64_t n2, cudaStream_t st);
cudaError_t launch_generate(const GenArgs& a, int uniform_th, cudaStream_t st);
cudaError_t launch_plan(const PlanArgs& a, cudaStream_t st);
cudaError_t launch_hist(const HistArgs& a, cudaStream_t st);
cudaError_t launch_order(const OrderArgs& a, int sm_count, cudaStream_t st);
cudaError_t launch_selftest_log(const double* x, double* out_fast, double* out_ref, int64_t n,
                                cudaStream_t st);

}  // namespace evs

// extern "C" entry points of libevsim_b200.so (see include/evsim_b200.h).
//
// One evs_step = k_prologue (clock + counters; validation for calls of < 4
// frames) -> k_generate (K1, per-tile event regions) -> k_group_hist (t_rel
// histogram rows of the tile groups) -> k_tilescan (tile bases, counts,
// capacity, column scan of the rows) -> k_tile_order (K2: canonical order, or
// pixel-major compaction for the serial API) [-> generic onesweep passes when
// t_now - t_prev exceeds 2^11 us].
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/evsim_b200.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace evs;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

int sm_count_current() {
  int dev = 0;
  cudaGetDevice(&dev);
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

struct StepLayout {
  int nseg, ntiles, npass, bits, NB, ngroups, gt, rows_stride, tile_px, tile_cap;
  int64_t max_tiles2, ovf_lim, ovf_cap, n2;
  size_t chunk_flag;
  size_t ctr, desc, zero2, region, tile_count, tile_ovf, tile_base, ovf_area, rows, tot, hist, gstart,
      seg_tbase, seg_dt, seg_tile_prefix, status2, keysA, keysB, total, bak_ref, bak_last, snap_ref, snap_last;
};

__global__ void k_clock_init(StepDesc* d, int64_t t0, uint32_t epoch) {
  d->next_t0 = t0;
  d->cur_t0 = t0;
  d->next_epoch = epoch;
  d->cur_epoch = epoch;
}

bool step_layout(const evs_step_params* p, StepLayout* L) {
  if (!p || p->streams < 1 || p->frames < 1 || p->height < 1 || p->width < 1) return false;
  if (p->height > 65535 || p->width > 65535 || p->capacity < 0) return false;
  const int64_t P = (int64_t)p->height * p->width;
  L->nseg = p->streams * p->frames;
  // K1 tiles: 1024 pixels (4 per thread); a batch too small to fill the GPU
  // with them (one small sensor) gets 256-pixel tiles (one pixel per thread):
  // 4x more CTAs and warps over the same pixels
  {
    const int64_t big = (int64_t)p->streams * ((P + kGenTile - 1) / kGenTile);
    L->tile_px = big < 2 * (int64_t)sm_count_current() ? kGenTile / kGenVpt : kGenTile;
    L->tile_cap = 4 * L->tile_px;
  }
  L->ntiles = (int)((P + L->tile_px - 1) / L->tile_px);
  const bool canon = p->order == EVS_ORDER_CANONICAL;
  int tbits = 1;
  if (canon) {
    const int64_t mdt = p->max_dt > 0 ? p->max_dt : p->tick;
    if (mdt <= 0 || mdt >= (1ll << 31)) return false;
    tbits = ilog2_ceil((uint64_t)mdt);
    if (tbits < 1) tbits = 1;
  }
  L->npass = canon ? (tbits + kMaxDigitBits - 1) / kMaxDigitBits : 0;
  L->bits = canon ? (tbits + L->npass - 1) / L->npass : 0;
  L->NB = canon ? (1 << L->bits) : 0;
  L->max_tiles2 = (canon && L->npass > 1) ? (p->capacity + kOrdTile - 1) / kOrdTile : 0;
  // tiles per histogram row / K2 CTA: as large as possible (fewer rows, longer
  // K2 chunks) while keeping >= 1.5 K2 CTAs per SM over the whole batch (a
  // single HD frame: 4 tiles -> 225 CTAs, inside one wave of 3 per SM)
  {
    const int64_t want = 3 * (int64_t)sm_count_current() / 2;
    L->gt = 1;
    for (int g = kMaxGroupTiles; g > 1; --g)
      if ((int64_t)((L->ntiles + g - 1) / g) * L->nseg >= want) { L->gt = g; break; }
  }
  // a call of many K2 CTAs (>= 8 waves at the largest groups) may use groups
  // down to half that size when the caller expects dense frames (keys_hint:
  // one K2 chunk of keys per group -- each chunk pays K2's per-bin column
  // prefix, scan and barriers, and one-chunk CTAs turn over fastest; HD T=50:
  // K2 0.429 -> 0.399 ms with 8-tile groups, while a sparse DAVIS stream is
  // slower with them).  The rows are always stored for the smallest choice,
  // so the workspace does not depend on the hint.
  int gt_min = L->gt;
  if ((int64_t)((L->ntiles + L->gt - 1) / L->gt) * L->nseg >= 16 * (int64_t)sm_count_current())
    gt_min = L->gt / 2 > 1 ? L->gt / 2 : 1;
  L->rows_stride = (L->ntiles + gt_min - 1) / gt_min;
  if (p->keys_hint > 0 && gt_min < L->gt) {
    const int64_t per_chunk = tile_order_chunk_keys(L->tile_px, canon ? 0 : 1, L->bits);
    const int64_t g = per_chunk * L->ntiles / p->keys_hint;  // tiles whose mean keys fill one chunk
    L->gt = (int)(g < gt_min ? gt_min : (g > L->gt ? L->gt : g));
  }
  L->ngroups = (L->ntiles + L->gt - 1) / L->gt;
  // spill area per segment: [0, ovf_lim) is claimed by K1 tiles whose keys do
  // not fit their region (atomic cursor, arrival order); a tile that finds it
  // full keeps only its count and a pre-frame state snapshot, and k_group_hist
  // regenerates it into [ovf_lim, ovf_lim + capacity) when it lies inside the
  // kept prefix (the kept events of a frame never exceed the capacity)
  L->ovf_lim = (int64_t)L->tile_cap * (1 + L->ntiles / 4);
  L->ovf_cap = L->ovf_lim + p->capacity;
  const size_t ns = (size_t)L->nseg, nt = (size_t)L->ntiles;
  size_t off = 0;
  L->ctr = off; off = align_up(off + 64 * sizeof(uint32_t));
  L->desc = off; off = align_up(off + sizeof(StepDesc));
  // zeroed by the prologue: spill cursors [nseg], K1 error word, K1 CTA ticket
  L->n2 = (int64_t)ns + 2;
  L->zero2 = off; off = align_up(off + (size_t)L->n2 * 8);
  L->chunk_flag = off; off = align_up(off + (size_t)p->streams * nt * 8);
  L->tile_count = off; off = align_up(off + ns * nt * 8);
  L->tile_ovf = off; off = align_up(off + ns * nt * 8);
  L->tile_base = off; off = align_up(off + ns * nt * 8);
  L->seg_tbase = off; off = align_up(off + ns * 8);
  L->seg_dt = off; off = align_up(off + ns * 8);
  L->rows = off; off = align_up(off + (canon ? ns * L->rows_stride * L->NB * 4 : 0));
  L->tot = off; off = align_up(off + ns * L->NB * 4);
  L->hist = off; off = align_up(off + (L->npass > 1 ? ns * L->npass * kHistReps * L->NB * 4 : 0));
  L->gstart = off; off = align_up(off + ns * L->NB * 4);
  L->seg_tile_prefix = off; off = align_up(off + (ns + 1) * 4);
  L->status2 = off; off = align_up(off + ns * L->max_tiles2 * L->NB * 8);
  L->keysA = off; off = align_up(off + (canon && L->npass > 1 ? ns * p->capacity * 8 : 0));
  L->keysB = off; off = align_up(off + (canon && L->npass > 1 ? ns * p->capacity * 8 : 0));
  const bool bak = p->frames >= 4;  // fused validation (step_impl)
  L->bak_ref = off; off = align_up(off + (bak ? (size_t)p->streams * P * 4 : 0));
  L->bak_last = off; off = align_up(off + (bak ? (size_t)p->streams * P * 8 : 0));
  L->region = off; off = align_up(off + ns * nt * L->tile_cap * 8);
  L->ovf_area = off; off = align_up(off + ns * (size_t)L->ovf_cap * 8);
  L->snap_ref = off; off = align_up(off + ns * nt * L->tile_px * 4);
  L->snap_last = off; off = align_up(off + ns * nt * L->tile_px * 4);
  L->total = off;
  return true;
}

template <typename T>
T* at(void* ws, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(ws) + off); }

}  // namespace

extern "C" {

int evs_version(void) { return 2; }

const char* evs_error_string(evs_status code) {
  switch (code) {
    case EVS_OK: return "ok";
    case EVS_ERR_ARG: return "invalid argument";
    case EVS_ERR_CUDA: return "CUDA error";
    case EVS_ERR_WORKSPACE: return "workspace too small";
    case EVS_ERR_UNSUPPORTED: return "unsupported input";
    default: return "unknown error";
  }
}

size_t evs_step_workspace_bytes(const evs_step_params* p) {
  StepLayout L;
  if (!step_layout(p, &L)) return 0;
  return L.total;
}

static evs_status step_impl(const evs_step_params* p, const evs_step_buffers* b, void* ws,
                            size_t ws_bytes, void* stream, void* const* evs, int nev) {
  StepLayout L;
  if (!step_layout(p, &L) || !b) return EVS_ERR_ARG;
  // refractory periods are compared in int32 against last-event times clamped
  // to [-2^30, 2^30] relative to the frame start: exact for refractory < 2^30 us
  if (p->log_eps <= 0 || p->refractory_us < 0 || p->refractory_us >= (1ll << 30) || p->capacity >= (1ll << 32))
    return EVS_ERR_ARG;
  if (!b->frames || !b->ref_log || !b->last_event_t || !b->counts || !b->dropped ||
      !b->reservations || !b->bad_pixel)
    return EVS_ERR_ARG;
  if (!b->t_bounds && (p->tick <= 0 || p->tick >= (1ll << 31))) return EVS_ERR_ARG;
  if ((b->th_pos == nullptr) != (b->th_neg == nullptr)) return EVS_ERR_ARG;
  if (!ws || ws_bytes < L.total) return EVS_ERR_WORKSPACE;
  const bool dclock = (p->flags & EVS_FLAG_DEVICE_CLOCK) != 0;
  if (!dclock && (p->epoch == 0 || p->epoch + EVS_EPOCHS_PER_CALL > EVS_EPOCH_LIMIT)) return EVS_ERR_ARG;
  if (dclock && b->t_bounds) return EVS_ERR_ARG;
  StepDesc* desc = dclock ? at<StepDesc>(ws, L.desc) : nullptr;
  const bool canon = p->order == EVS_ORDER_CANONICAL;
  if (p->capacity > 0 && (!b->ev_t || !b->ev_x || !b->ev_y || !b->ev_p)) return EVS_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t P = (int64_t)p->height * p->width;
  auto mark = [&](int i) {
    if (evs && i < nev && evs[i]) cudaEventRecord(static_cast<cudaEvent_t>(evs[i]), st);
  };
  int64_t* zero2 = at<int64_t>(ws, L.zero2);

  mark(0);
  // the tile-order path validates inside K1 (fused: K1 backs up the state it
  // overwrites, 12 B/px) when the call has >= 4 frames per stream; shorter calls
  // read the frames once in the prologue (4 B/px per frame) instead
  const bool fuse_val = p->validate && p->frames >= 4;
  cudaError_t e = launch_prologue(b->frames, (int64_t)L.nseg * P, P, fuse_val ? 0 : p->validate, b->bad_pixel,
                                  b->reservations, L.nseg, desc,
                                  (int64_t)p->frames * p->tick * (p->clock_stride > 1 ? p->clock_stride : 1), zero2,
                                  L.n2, st);
  if (e != cudaSuccess) return EVS_ERR_CUDA;
  mark(1);

  GenArgs g;
  memset(&g, 0, sizeof(g));
  g.S = p->streams; g.T = p->frames; g.H = p->height; g.W = p->width; g.P = P;
  g.log_eps = p->log_eps; g.log_eps_f = (float)p->log_eps;
  g.refr = p->refractory_us; g.cap = p->capacity;
  g.thp_u = p->th_pos_uniform; g.thn_u = p->th_neg_uniform;
  g.frames = b->frames; g.t_bounds = b->t_bounds; g.t0 = p->t0; g.tick = p->tick;
  g.max_dt = p->max_dt > 0 ? p->max_dt : p->tick;
  g.ref = b->ref_log; g.last = b->last_event_t; g.thp = b->th_pos; g.thn = b->th_neg;
  g.seg_res = b->reservations;
  g.seg_tbase = at<int64_t>(ws, L.seg_tbase);
  g.hist_bits = L.bits;
  g.bad = b->bad_pixel;
  g.epoch = p->epoch;
  g.ntiles = L.ntiles;
  g.tile_px = L.tile_px; g.tile_cap = L.tile_cap;
  g.desc = desc;
  g.rows = canon ? at<uint32_t>(ws, L.rows) : nullptr;
  g.ngroups = L.ngroups;
  g.gt = L.gt;
  {
    // split each tile's T frames into chunks so the grid is >= ~8 waves of
    // resident K1 CTAs (4 per SM; HD T=50: 6 chunks of 9 frames, measured best
    // against 4, 5 and 8): the tail wave then lasts one short chunk
    const int64_t resident = (int64_t)sm_count_current() * 4;
    const int64_t tiles = (int64_t)p->streams * L.ntiles;
    int64_t nch = (8 * resident + tiles - 1) / tiles;
    // >= 2 frames per chunk: one-frame chunks of a small sensor serialise on
    // the chunk hand-off (DAVIS T=50: 50 chunks ran 17 % slower than 25)
    if (nch > (p->frames + 1) / 2) nch = (p->frames + 1) / 2;
    if (nch > 255) nch = 255;
    if (nch < 1) nch = 1;
    g.tc = (int)((p->frames + nch - 1) / nch);
    g.nchunks = (p->frames + g.tc - 1) / g.tc;
    g.chunk_flag = at<unsigned long long>(ws, L.chunk_flag);
  }
  g.region = at<uint64_t>(ws, L.region);
  g.tile_count = at<int64_t>(ws, L.tile_count);
  g.tile_ovf = at<int64_t>(ws, L.tile_ovf);
  g.ovf_area = at<uint64_t>(ws, L.ovf_area);
  g.ovf_cursor = reinterpret_cast<unsigned long long*>(zero2);
  g.ovf_cap = L.ovf_cap;
  g.ovf_lim = L.ovf_lim;
  g.err = zero2 + L.nseg;
  g.ticket = reinterpret_cast<unsigned int*>(zero2 + L.nseg + 1);
  g.seg_dt = at<int64_t>(ws, L.seg_dt);
  g.snap_ref = at<float>(ws, L.snap_ref);
  g.snap_last = at<int32_t>(ws, L.snap_last);
  g.fuse_validate = fuse_val ? 1 : 0;
  g.bad_rw = b->bad_pixel;
  g.bak_ref = at<float>(ws, L.bak_ref);
  g.bak_last = at<int64_t>(ws, L.bak_last);
  e = launch_generate(g, b->th_pos == nullptr, st);
  if (e != cudaSuccess) return EVS_ERR_CUDA;
  mark(2);

  TileScanArgs ts;
  memset(&ts, 0, sizeof(ts));
  ts.tile_px = L.tile_px; ts.tile_cap = L.tile_cap;
  ts.nseg = L.nseg; ts.ntiles = L.ntiles; ts.ngroups = L.ngroups; ts.bits = L.bits; ts.cap = p->capacity;
  ts.gt = L.gt;
  ts.rows_stride = L.rows_stride;
  ts.tile_count = g.tile_count; ts.tile_ovf = g.tile_ovf; ts.region = g.region; ts.ovf_area = g.ovf_area;
  ts.ovf_cap = L.ovf_cap; ts.tile_base = at<int64_t>(ws, L.tile_base);
  // regeneration of the tiles K1 could not store (k_group_hist)
  ts.ovf_lim = L.ovf_lim; ts.ovf_cursor = g.ovf_cursor; ts.err_rw = g.err;
  ts.frames = b->frames; ts.T = p->frames; ts.W = p->width; ts.P = P;
  ts.thp = b->th_pos; ts.thn = b->th_neg; ts.thp_u = p->th_pos_uniform; ts.thn_u = p->th_neg_uniform;
  ts.log_eps = p->log_eps; ts.refr = (int)p->refractory_us;
  ts.seg_tbase = g.seg_tbase; ts.seg_dt = g.seg_dt; ts.snap_ref = g.snap_ref; ts.snap_last = g.snap_last;
  ts.rows = g.rows; ts.tot = at<uint32_t>(ws, L.tot);
  ts.out_count = b->counts; ts.out_dropped = b->dropped; ts.bad = b->bad_pixel; ts.err = g.err;
  if (fuse_val) {
    ts.bak_ref = g.bak_ref; ts.bak_last = g.bak_last;
    ts.ref = b->ref_log; ts.last = b->last_event_t; ts.sp = (int64_t)p->streams * P;
  }
  // (pixel-major order: no histogram rows, only the regeneration of tiles K1
  // could not store)
  e = launch_group_hist(ts, st);
  if (e != cudaSuccess) return EVS_ERR_CUDA;
  e = launch_tilescan(ts, st);
  if (e != cudaSuccess) return EVS_ERR_CUDA;
  mark(3);

  TileOrderArgs to;
  memset(&to, 0, sizeof(to));
  to.tile_px = L.tile_px; to.tile_cap = L.tile_cap;
  to.nseg = L.nseg; to.ntiles = L.ntiles; to.ngroups = L.ngroups; to.bits = L.bits; to.shift = kKeyPixBits;
  to.gt = L.gt;
  to.rows_stride = L.rows_stride;
  to.cap = p->capacity; to.tile_count = g.tile_count; to.tile_ovf = g.tile_ovf; to.tile_base = ts.tile_base;
  to.region = g.region; to.ovf_area = g.ovf_area; to.ovf_cap = L.ovf_cap; to.rows = g.rows; to.tot = ts.tot;
  to.seg_stride = p->capacity; to.pixel_major = canon ? 0 : 1;
  to.final_soa = (!canon || L.npass == 1) ? 1 : 0;
  to.keys_out = at<uint64_t>(ws, L.keysB);
  to.out_t = b->ev_t; to.out_x = b->ev_x; to.out_y = b->ev_y; to.out_p = b->ev_p;
  to.seg_tbase = g.seg_tbase; to.bad = b->bad_pixel;
  e = launch_tile_order(to, st);
  if (e != cudaSuccess) return EVS_ERR_CUDA;

  if (canon && L.npass > 1) {
    // wide t_rel (dt > 2^11 us): remaining digits with generic onesweep passes
    HistArgs h;
    h.nseg = L.nseg; h.keys = to.keys_out; h.seg_stride = p->capacity; h.seg_count = b->counts;
    h.npass = L.npass; h.pass0 = 1; h.bits = L.bits; h.base_shift = kKeyPixBits;
    h.hist = at<uint32_t>(ws, L.hist);
    e = launch_hist(h, st);
    if (e != cudaSuccess) return EVS_ERR_CUDA;
    const int sms = sm_count_current();
    for (int pass = 1; pass < L.npass; ++pass) {
      PlanArgs pl;
      memset(&pl, 0, sizeof(pl));
      pl.nseg = L.nseg; pl.cap = p->capacity; pl.seg_total = b->counts;
      pl.hist = h.hist; pl.npass = L.npass; pl.pass = pass; pl.bits = L.bits;
      pl.gstart = at<uint32_t>(ws, L.gstart);
      pl.seg_tile_prefix = at<uint32_t>(ws, L.seg_tile_prefix);
      pl.bad = b->bad_pixel; pl.zero_hist = 1;
      e = launch_plan(pl, st);
      if (e != cudaSuccess) return EVS_ERR_CUDA;
      OrderArgs o;
      memset(&o, 0, sizeof(o));
      o.nseg = L.nseg;
      o.keys_in = (pass % 2 == 1) ? at<uint64_t>(ws, L.keysB) : at<uint64_t>(ws, L.keysA);
      o.keys_out = (pass % 2 == 1) ? at<uint64_t>(ws, L.keysA) : at<uint64_t>(ws, L.keysB);
      o.seg_stride = p->capacity; o.seg_count = b->counts;
      o.seg_tile_prefix = pl.seg_tile_prefix;
      o.gstart = pl.gstart; o.shift = kKeyPixBits + pass * L.bits; o.bits = L.bits;
      o.status = at<uint64_t>(ws, L.status2); o.max_tiles = L.max_tiles2;
      o.ctr = at<uint32_t>(ws, L.ctr) + 1 + pass;
      o.epoch = dclock ? (uint32_t)(1 + pass) : p->epoch + 1 + pass;
      o.desc = desc;
      o.final_soa = pass == L.npass - 1;
      o.out_t = b->ev_t; o.out_x = b->ev_x; o.out_y = b->ev_y; o.out_p = b->ev_p;
      o.seg_tbase = g.seg_tbase;
      e = launch_order(o, sms, st);
      if (e != cudaSuccess) return EVS_ERR_CUDA;
    }
  }
  mark(4);
  return EVS_OK;
}

evs_status evs_step(const evs_step_params* p, const evs_step_buffers* b, void* ws, size_t ws_bytes,
                    void* stream) {
  return step_impl(p, b, ws, ws_bytes, stream, nullptr, 0);
}

evs_status evs_step_profiled(const evs_step_params* p, const evs_step_buffers* b, void* ws,
                             size_t ws_bytes, void* stream, void* const* stage_events,
                             int32_t n_events) {
  return step_impl(p, b, ws, ws_bytes, stream, stage_events, n_events);
}

evs_status evs_selftest_log(int64_t n, const double* x, double* out_fast, double* out_cuda, void* stream) {
  if (n < 0 || (n > 0 && (!x || !out_fast || !out_cuda))) return EVS_ERR_ARG;
  return launch_selftest_log(x, out_fast, out_cuda, n, static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? EVS_OK : EVS_ERR_CUDA;
}

static void step_regions(const evs_step_params* p, const evs_step_buffers* b, const StepLayout& L, const void* ws,
                         StepVoxArgs* a) {
  memset(a, 0, sizeof(*a));
  a->ntiles = L.ntiles; a->T = p->frames; a->W = p->width;
  a->tile_px = L.tile_px; a->tile_cap = L.tile_cap;
  a->P = (int64_t)p->height * p->width; a->cap = p->capacity; a->ovf_cap = L.ovf_cap;
  void* w = const_cast<void*>(ws);
  a->tile_count = at<int64_t>(w, L.tile_count);
  a->tile_base = at<int64_t>(w, L.tile_base);
  a->tile_ovf = at<int64_t>(w, L.tile_ovf);
  a->region = at<uint64_t>(w, L.region);
  a->ovf_area = at<uint64_t>(w, L.ovf_area);
  a->seg_tbase = at<int64_t>(w, L.seg_tbase);
  a->bad = b->bad_pixel;
}

evs_status evs_step_voxel(const evs_step_params* p, const evs_step_buffers* b, const void* ws, size_t ws_bytes,
                          int32_t stream_index, int64_t t0, int64_t t1, int32_t bins, int32_t flags, float* out,
                          void* voxel_ws, size_t voxel_ws_bytes, void* stream) {
  StepLayout L;
  if (!step_layout(p, &L) || !b || !b->bad_pixel) return EVS_ERR_ARG;
  if (!ws || ws_bytes < L.total) return EVS_ERR_WORKSPACE;
  if (stream_index < 0 || stream_index >= p->streams || t1 <= t0 || bins < 2 || bins > kStepVoxMaxBins)
    return EVS_ERR_ARG;
  const int64_t P = (int64_t)p->height * p->width;
  const bool fin = (flags & EVS_VOXEL_FINALIZE) != 0;
  if (fin ? !out : (!voxel_ws || voxel_ws_bytes < (size_t)bins * P * sizeof(long long))) return EVS_ERR_ARG;
  StepVoxArgs a;
  step_regions(p, b, L, ws, &a);
  a.s = stream_index; a.B = bins;
  a.t0 = t0; a.t1 = t1;
  a.out = fin ? out : nullptr;
  a.acc_out = fin ? nullptr : static_cast<long long*>(voxel_ws);
  return launch_step_voxel(a, static_cast<cudaStream_t>(stream)) == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

evs_status evs_step_histogram(const evs_step_params* p, const evs_step_buffers* b, const void* ws,
                              size_t ws_bytes, int64_t window_us, int64_t t_end, int64_t* out, void* stream) {
  StepLayout L;
  if (!step_layout(p, &L) || !b || !b->bad_pixel || !out) return EVS_ERR_ARG;
  if (!ws || ws_bytes < L.total) return EVS_ERR_WORKSPACE;
  if (p->streams > 65535) return EVS_ERR_ARG;
  StepVoxArgs a;
  step_regions(p, b, L, ws, &a);
  return launch_step_hist(a, p->streams, t_end - window_us, t_end, out, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

evs_status evs_step_clock_init(const evs_step_params* p, void* ws, size_t ws_bytes, int64_t t0,
                               uint32_t epoch, void* stream) {
  StepLayout L;
  if (!step_layout(p, &L)) return EVS_ERR_ARG;
  if (!ws || ws_bytes < L.total) return EVS_ERR_WORKSPACE;
  if (epoch == 0 || epoch + EVS_EPOCHS_PER_CALL > EVS_EPOCH_LIMIT) return EVS_ERR_ARG;
  k_clock_init<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(at<StepDesc>(ws, L.desc), t0, epoch);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

}  // extern "C"

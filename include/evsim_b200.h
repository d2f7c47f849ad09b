/*
 * evsim_b200.h -- C ABI of the B200-native event-camera hot path.
 *
 * Drop-in boundary for the reference's in-process event API
 * (/root/reference/pkg/src/evsim/events/__init__.py:3-57).  Every entry
 * point takes plain device pointers and sizes, is asynchronous on the given
 * CUDA stream (a cudaStream_t passed as void*; NULL = legacy default
 * stream), and returns an evs_status.  No torch types cross this boundary.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src):
 *   evs_step            generate_events_parallel  evsim/events/parallel.py:126-273
 *                       generate_events_serial    evsim/events/model.py:79-171
 *                       (+ canonical_sort of the result, parallel.py:112-123,
 *                        and log_transform validation, model.py:28-39)
 *   evs_canonical_sort  canonical_sort            evsim/events/parallel.py:112-123
 *   evs_noise           inject_noise_events       evsim/events/model.py:174-212
 *   evs_noise_batch     the same for the frames of a window, batched launches
 *   evs_accumulate      accumulate_events_to_image evsim/events/model.py:249-262
 *   evs_voxel           (no reference counterpart; repo-defined voxel grid)
 *   evs_voxel_segments  the same over many device-counted segments (a window)
 *   evs_step_voxel      the same from a step's per-tile regions (no atomics)
 *   evs_step_histogram  accumulate_events_to_image of every stream of a step
 *   evs_compact_segments packs a step's segments back to back (one D2H per array)
 *   evs_limit_bandwidth limit_bandwidth           evsim/events/model.py:215-246
 *   evs_render          render_pair               evsim/render.py:179-208 (frame producer)
 *   evs_seed_pcg64      numpy default_rng(seed) seeding used by
 *                       inject_noise_events (model.py:194) -- host only
 */
#ifndef EVSIM_B200_H
#define EVSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int evs_status;
#define EVS_OK 0
#define EVS_ERR_ARG 1       /* invalid argument (reference ValueError class) */
#define EVS_ERR_CUDA 2      /* CUDA launch / runtime failure */
#define EVS_ERR_WORKSPACE 3 /* workspace too small */
#define EVS_ERR_UNSUPPORTED 4

#define EVS_ORDER_PIXEL_MAJOR 0 /* generate_events_serial order (model.py:140-158) */
#define EVS_ORDER_CANONICAL 1   /* (t, y, x, p) ascending (parallel.py:116) */

/* Each evs_step call consumes this many consecutive epoch values. */
#define EVS_EPOCHS_PER_CALL 8u
/* Epochs are 22-bit; when epoch + EVS_EPOCHS_PER_CALL would exceed this,
 * zero the workspace and restart the caller's counter at 1. */
#define EVS_EPOCH_LIMIT ((1u << 22) - 1u)

/* EventCameraConfig (types.py:129-156) + batch shape of one evs_step call:
 * S independent sensors ("streams"), T consecutive frames per sensor. */
typedef struct evs_step_params {
  int32_t streams;       /* S >= 1 */
  int32_t frames;        /* T >= 1 */
  int32_t height;        /* H (<= 65535) */
  int32_t width;         /* W (<= 65535) */
  double log_eps;        /* > 0 */
  int64_t refractory_us; /* >= 0 */
  int64_t capacity;      /* max events kept per (stream, frame); output stride */
  float th_pos_uniform;  /* used when th_pos == NULL (sigma_c == 0) */
  float th_neg_uniform;
  int64_t t0;            /* when t_bounds == NULL: frame f spans [t0+f*tick, t0+(f+1)*tick) */
  int64_t tick;
  int64_t max_dt;        /* upper bound of t_now - t_prev over the call (< 2^31) */
  int32_t order;         /* EVS_ORDER_* */
  int32_t validate;      /* 1: reject invalid frames before touching state */
  uint32_t epoch;        /* caller-maintained counter, see EVS_EPOCHS_PER_CALL */
  int32_t flags;         /* EVS_FLAG_* */
  int32_t clock_stride;  /* device clock: steps of this workspace are clock_stride calls apart (0/1:
                            consecutive; 2: two engines alternating, see evs_step_clock_init) */
  int64_t keys_hint;     /* expected events per (stream, frame), e.g. the previous call's mean
                            (0: none).  Performance only: it sizes the tile groups of the
                            ordering pass (the workspace does not depend on it); results are
                            identical for any value */
} evs_step_params;

/* flags: t0 and epoch are taken from a clock kept in the workspace and
 * advanced on the device by every step (t0 += frames*tick, epoch += 8), so a
 * captured CUDA graph of evs_step calls can be replayed.  Initialise it with
 * evs_step_clock_init; params.t0 / params.epoch are then ignored. */
#define EVS_FLAG_DEVICE_CLOCK 1

/* Device buffers of one evs_step call.  Segment g = s*T + f. */
typedef struct evs_step_buffers {
  const float* frames;     /* [S][T][H*W] intensities in [0,1] */
  const int64_t* t_bounds; /* [S][T+1] frame timestamps (us) or NULL (t0/tick) */
  float* ref_log;          /* [S][H*W] in/out (PixelStateGrid.ref_log) */
  int64_t* last_event_t;   /* [S][H*W] in/out (PixelStateGrid.last_event_t) */
  const float* th_pos;     /* [S][H*W] or NULL (uniform) */
  const float* th_neg;     /* [S][H*W] or NULL (uniform) */
  int64_t* ev_t;           /* [S*T][capacity] event time (us) */
  uint16_t* ev_x;          /* [S*T][capacity] */
  uint16_t* ev_y;          /* [S*T][capacity] */
  int8_t* ev_p;            /* [S*T][capacity] polarity +1/-1 */
  int64_t* counts;         /* [S*T] events written (= min(kept, capacity)) */
  int64_t* dropped;        /* [S*T] EventBatch.dropped_count (events beyond the capacity); -2: a
                              pixel would cross > 2^20 thresholds in one frame (+inf intensity
                              without validation, or a corrupt ref_log) -- the call's outputs
                              are then invalid */
  int64_t* reservations;   /* [S*T] AggregationStats.reservation_count */
  int64_t* bad_pixel;      /* [1] must hold INT64_MAX on entry; receives the first
                              invalid flat index into frames (s*T*H*W + f*H*W + i) */
} evs_step_buffers;

int evs_version(void);
const char* evs_error_string(evs_status code);
/* Bytes of device workspace evs_step needs for these params (zero-filled
 * once by the caller; reusable across calls with the same params). */
size_t evs_step_workspace_bytes(const evs_step_params* p);
evs_status evs_step(const evs_step_params* p, const evs_step_buffers* b, void* workspace,
                    size_t workspace_bytes, void* stream);
/* Set the device clock of a workspace (EVS_FLAG_DEVICE_CLOCK): the next step
 * starts at t0 and uses epoch (asynchronous on stream). */
evs_status evs_step_clock_init(const evs_step_params* p, void* workspace, size_t workspace_bytes,
                               int64_t t0, uint32_t epoch, void* stream);

/* evs_step that also records stage_events[i] (cudaEvent_t handles; NULL
 * entries skipped) on `stream`: [0] before the validation prologue,
 * [1] after it, [2] after the fused generate kernel, [3] after planning,
 * [4] after the ordering pass(es).  Used for per-kernel roofline timing. */
evs_status evs_step_profiled(const evs_step_params* p, const evs_step_buffers* b, void* workspace,
                             size_t workspace_bytes, void* stream, void* const* stage_events,
                             int32_t n_events);

/* canonical_sort of one device batch of n events, in place.  Requires
 * polarity in {-1,+1} and max(t)-min(t) < 2^31.  Workspace from
 * evs_sort_workspace_bytes(n).  t_min/t_span from the caller (host). */
size_t evs_sort_workspace_bytes(int64_t n, int64_t t_span);
evs_status evs_canonical_sort(int64_t n, int64_t* t, uint16_t* x, uint16_t* y, int8_t* p,
                              int64_t t_min, int64_t t_span, uint32_t epoch, void* workspace,
                              size_t workspace_bytes, void* stream);
/* canonical_sort (parallel.py:112-123) of ANY device batch of n < 2^32 events,
 * in place: t compared as uint64 (any span, values >= 2^63 included), any
 * int8 polarity (signed order), stable.  Four LSD passes over 32-bit digits
 * (polarity, (y, x), t low word, t high word), each a radix sort of 64-bit
 * keys digit << 32 | position.  Workspace from evs_sort_general_workspace_bytes. */
size_t evs_sort_general_workspace_bytes(int64_t n);
evs_status evs_canonical_sort_general(int64_t n, int64_t* t, uint16_t* x, uint16_t* y, int8_t* p,
                                      void* workspace, size_t workspace_bytes, void* stream);
/* Stable merge of two canonical-ordered device batches A (signal) and B
 * (noise) into out[na + nb]: the canonical order of concat_batches([A, B])
 * (types.py:82-92 then parallel.py:112-123) without a full sort.  Requires
 * t >= t_min, t - t_min < 2^31 and polarity in {-1,+1}; workspace >= nb*8 B. */
evs_status evs_merge_canonical(int64_t na, const int64_t* at, const uint16_t* ax, const uint16_t* ay,
                               const int8_t* ap, int64_t nb, const int64_t* bt, const uint16_t* bx,
                               const uint16_t* by, const int8_t* bp, int64_t t_min, int64_t* out_t,
                               uint16_t* out_x, uint16_t* out_y, int8_t* out_p, void* workspace,
                               size_t workspace_bytes, void* stream);
/* batch statistics used to choose the sort path: out[0]=min t, out[1]=max t,
 * out[2]=max x, out[3]=max y, out[4]=1 if any polarity not in {-1,+1}. */
evs_status evs_batch_stats(int64_t n, const int64_t* t, const uint16_t* x, const uint16_t* y,
                           const int8_t* p, int64_t* out5, void* stream);

/* Background noise (inject_noise_events, model.py:174-212), bit-exact with
 * numpy's Generator(PCG64(SeedSequence(seed))) draw order.  The caller
 * computes lam = rate * (dt * 1e-6) and enlam = exp(-lam) on the host (as
 * numpy does) and the PCG64 state with evs_seed_pcg64. */
typedef struct evs_noise_params {
  int32_t width, height;
  int64_t t_prev, t_now;
  double lam;         /* > 0 */
  double enlam;       /* exp(-lam) */
  uint64_t pcg[4];    /* state_hi, state_lo, inc_hi, inc_lo */
  int64_t capacity;   /* event capacity; 0 = automatic (mean + 12 sigma) */
  int32_t order;      /* 0: reference order -> ev_t/x/y/p; 1: (pixel, p, t) keys -> ev_key */
  uint32_t reserved;
  double draw_scale;  /* >= 1; enlarge the walked draw range (retry when meta[2] != 0) */
} evs_noise_params;
size_t evs_noise_workspace_bytes(const evs_noise_params* p);
/* capacity the call will use (host) */
int64_t evs_noise_capacity(const evs_noise_params* p);
/* meta_out (device, 4 x int64): [0] draws consumed by the counts, [1] events,
 * [2] != 0: draw range too short (retry with larger draw_scale),
 * [3] != 0: events exceed capacity (retry with larger capacity). */
evs_status evs_noise(const evs_noise_params* p, int64_t* ev_t, uint16_t* ev_x, uint16_t* ev_y,
                     int8_t* ev_p, uint64_t* ev_key, int64_t* meta_out, void* workspace,
                     size_t workspace_bytes, void* stream);

/* evs_noise for nf frames at once (e.g. the ticks of one window), batched
 * kernel launches: frame f's events go to row f (element offset f*ev_stride,
 * ev_stride >= that frame's evs_noise_capacity; order 0 only) and its meta to
 * meta_out[4f..4f+3] (same meaning as evs_noise; a flagged frame is redone by
 * the caller with evs_noise).  Workspace: evs_noise_batch_workspace_bytes. */
size_t evs_noise_batch_workspace_bytes(const evs_noise_params* ps, int32_t nf);
evs_status evs_noise_batch(const evs_noise_params* ps, int32_t nf, int64_t* ev_t, uint16_t* ev_x, uint16_t* ev_y,
                           int8_t* ev_p, int64_t ev_stride, int64_t* meta_out, void* workspace,
                           size_t workspace_bytes, void* stream);

/* accumulate_events_to_image (model.py:249-262) of a device batch into an
 * int64 (H, W) grid; the caller checks coordinate bounds first (ValueError,
 * model.py:253-254, see evs_batch_stats). */
evs_status evs_accumulate(int64_t n, const int64_t* t, const uint16_t* x, const uint16_t* y,
                          const int8_t* p, int64_t window_us, int64_t t_end, int32_t width,
                          int32_t height, int64_t* grid, void* stream);

/* Voxel grid (no reference counterpart): out[b][y][x]
 * = sum over events with t in [t0, t1) of p * max(0, D - |b*D - (B-1)(t-t0)|) / D,
 * D = t1 - t0, accumulated exactly in int64, rounded once to f32. */
size_t evs_voxel_workspace_bytes(int32_t bins, int32_t width, int32_t height);
evs_status evs_voxel(int64_t n, const int64_t* t, const uint16_t* x, const uint16_t* y,
                     const int8_t* p, int64_t t0, int64_t t1, int32_t bins, int32_t width,
                     int32_t height, float* out, void* workspace, size_t workspace_bytes,
                     void* stream);

/* The same voxel grid over many event segments without a host round trip:
 * segment s (s < nseg) holds counts[s * counts_stride] events (device int64)
 * at element offset s * seg_stride of t/x/y/p -- the S x T rows of an evs_step
 * output (counts = evs_step_buffers.counts, stride 1, seg_stride = capacity)
 * or per-frame noise buffers (counts = meta[1], stride 4).  flags:
 * EVS_VOXEL_CLEAR zeroes the int64 workspace first, EVS_VOXEL_FINALIZE rounds
 * it into out; calls in between accumulate (signal + noise of one window). */
#define EVS_VOXEL_CLEAR 1
#define EVS_VOXEL_FINALIZE 2
evs_status evs_voxel_segments(int32_t nseg, const int64_t* counts, int64_t counts_stride, int64_t seg_stride,
                              const int64_t* t, const uint16_t* x, const uint16_t* y, const int8_t* p,
                              int64_t t0, int64_t t1, int32_t bins, int32_t width, int32_t height,
                              int32_t flags, float* out, void* workspace, size_t workspace_bytes,
                              void* stream);

/* Voxel grid of stream `stream_index` over [t0, t1) from the events of the
 * last evs_step call made with these params / buffers / workspace (tile-order
 * path): read from the step's per-tile key regions, one CTA per 1024-pixel
 * tile accumulating its own pixels in shared memory (no global atomics).
 * flags & EVS_VOXEL_FINALIZE: the f32 grid goes to out; otherwise the int64
 * numerators are stored into voxel_ws (every pixel written: it replaces
 * EVS_VOXEL_CLEAR) for evs_voxel_segments to add noise and finalize.  bins <= 24.
 * EVS_ERR_UNSUPPORTED if the step ran the bucket path (EVS_PATH=bucket). */
evs_status evs_step_voxel(const evs_step_params* p, const evs_step_buffers* b, const void* workspace,
                          size_t workspace_bytes, int32_t stream_index, int64_t t0, int64_t t1, int32_t bins,
                          int32_t flags, float* out, void* voxel_ws, size_t voxel_ws_bytes, void* stream);

/* accumulate_events_to_image (model.py:249-262) of EVERY stream of the last
 * evs_step call on this workspace: out[s][y][x] (int64, device) = sum of the
 * polarities of stream s's events with t in [t_end - window_us, t_end), read
 * from the step's per-tile regions in one launch. */
evs_status evs_step_histogram(const evs_step_params* p, const evs_step_buffers* b, const void* workspace,
                              size_t workspace_bytes, int64_t window_us, int64_t t_end, int64_t* out,
                              void* stream);

/* Pack the first counts[g] (device int64) events of every segment g < nseg of
 * an evs_step output (stride seg_stride = capacity) back to back into out_*
 * (segment order), so a host copy is one transfer per array.  Nothing is
 * written at or beyond out_capacity elements (the caller compares the total). */
evs_status evs_compact_segments(int32_t nseg, const int64_t* counts, int64_t seg_stride, const int64_t* t,
                                const uint16_t* x, const uint16_t* y, const int8_t* p, int64_t* out_t,
                                uint16_t* out_x, uint16_t* out_y, int8_t* out_p, int64_t out_capacity,
                                void* stream);

/* Stable k-way merge of nruns <= 64 sorted runs of int64 keys stored back to
 * back in keys_in (run r = [run_offsets[r], run_offsets[r+1]), device int64)
 * into keys_out (ties keep run order).  The row bands of one sensor
 * are such runs of packed 8-byte keys whose integer order is
 * the canonical order (parallel.py:112-123): their merge is the sensor's
 * canonical batch. */
evs_status evs_merge_runs(int32_t nruns, const int64_t* run_offsets, int64_t n, const int64_t* keys_in,
                          int64_t* keys_out, void* stream);

/* Packed event keys of an evs_step output for a gather to one rank (SURVEY.md
 * 8(e); BASELINE config 5): the first counts[g] events of every segment
 * g < nseg (stride seg_stride) back to back, segment order, as
 *   key = (t - t_base) << (ybits + xbits + 1) | (y + y_offset) << (xbits + 1) | x << 1 | (p > 0)
 * in 4 bytes (key_bytes = 4: the key must fit 31 bits, e.g. DAVIS 12+9+9+1)
 * or 8 bytes (key_bytes = 8: t - t_base < 2^30, ybits = xbits = 16).  Integer
 * order of the keys within a segment is the canonical (t, y, x, p) order.
 * seg_offsets (device int64, nseg + 1) receives the exclusive prefix of the
 * counts and the total; nothing is written at or beyond out_capacity keys.
 * Replaces the host-side packing a consumer of parallel.py:112-123 output
 * would do before a transfer.  y_offset shifts a row band's rows to sensor rows. */
evs_status evs_pack_segments(int32_t nseg, const int64_t* counts, int64_t seg_stride, const int64_t* t,
                             const uint16_t* x, const uint16_t* y, const int8_t* p, int64_t t_base,
                             int32_t y_offset, int32_t key_bytes, int32_t ybits, int32_t xbits, void* out_keys,
                             int64_t* seg_offsets, int64_t out_capacity, void* stream);

/* limit_bandwidth (model.py:215-246) of a t-sorted device batch of n >= 1
 * events: keeps the first `cap` = int(rate * window * 1e-6) events of each
 * window tiling forward from t[0].  meta_out (device, 2 x int64): [0] kept
 * count, [1] != 0 if the batch is not t-sorted (reference ValueError). */
size_t evs_limit_bandwidth_workspace_bytes(int64_t n);
evs_status evs_limit_bandwidth(int64_t n, const int64_t* t, const uint16_t* x, const uint16_t* y,
                               const int8_t* p, int64_t cap, int64_t window_us, int64_t* out_t,
                               uint16_t* out_x, uint16_t* out_y, int8_t* out_p, int64_t* meta_out,
                               void* workspace, size_t workspace_bytes, void* stream);

/* Self-test of the kernels' table-driven f64 log (model.py:39 front-end):
 * out_fast[i] = the log used by evs_step, out_cuda[i] = CUDA's log(x[i]). */
evs_status evs_selftest_log(int64_t n, const double* x, double* out_fast, double* out_cuda,
                            void* stream);

/* log_transform (model.py:28-39) of n float32 intensities: out = log(double(v)
 * + log_eps) (f64, <= 1 ulp) and, in the same pass, the first invalid value
 * (not finite or outside [0, 1]) as a flat index in *bad_index (device int64,
 * the caller initialises it to INT64_MAX; atomicMin). */
evs_status evs_log_transform(int64_t n, const float* values, double log_eps, double* out, int64_t* bad_index,
                             void* stream);

/* numpy SeedSequence(seed) -> PCG64 state (host function, no GPU).
 * words: little-endian u32 words of the non-negative seed.
 * out: state_hi, state_lo, inc_hi, inc_lo. */
void evs_seed_pcg64(const uint32_t* words, int32_t nwords, uint64_t out[4]);


/* GPU frame producer: render_pair of the reference
 * (evsim/render.py:179-208) -- axis-aligned textured planes, pinhole camera,
 * projective z-depth, misses -> ambient intensity / +inf depth.  `planes` is a
 * DEVICE array; intensity / depth are device [H][W] f32 (depth may be NULL). */
#define EVS_TEX_CHECKER 0 /* Checkerboard(cell, intensity_a, intensity_b), render.py:60-74 */
#define EVS_TEX_NOISE 1   /* ValueNoise(scale, seed, lo, hi), render.py:78-108 */
typedef struct evs_plane {
  int32_t axis;      /* 0, 1, 2 */
  int32_t kind;      /* EVS_TEX_* */
  double offset;
  double bounds[4];  /* amin, amax, bmin, bmax over the other two axes (ascending index) */
  double cell;       /* checker cell size or noise scale */
  double value_a;    /* intensity_a or lo */
  double value_b;    /* intensity_b or hi */
  uint64_t seed;     /* noise seed */
} evs_plane;
typedef struct evs_render_params {
  int32_t width, height;
  double fx, fy, cx, cy;
  double rot[9];     /* world-from-body rotation, row-major (Pose.rotation_matrix) */
  double origin[3];  /* camera position */
  double ambient;
} evs_render_params;
evs_status evs_render(const evs_render_params* p, const evs_plane* planes, int32_t nplanes, float* intensity,
                      float* depth, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EVSIM_B200_H */

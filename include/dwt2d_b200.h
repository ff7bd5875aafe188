/*
 * dwt2d_b200 — C ABI of the B200-native 2-D DWT (arXiv 1704.08657 schemes).
 *
 * This is the drop-in boundary for the reference's transform path. The
 * reference exposes it as header-only C++ templates with no FFI
 * (reference: proj/include/dwt2d/executor.hpp:52-53 compile<T>, :196-197
 * run<T>, :242-244 inverse_lifting<T>; scheme.hpp:76-92 builders;
 * wavelet.hpp:37-45 wavelet lookup). Every entry point below replaces one of
 * those calls (cited per function); the C++ mirror of the reference API in
 * include/dwt2d_b200/executor.hpp is written on top of these functions.
 *
 * Conventions
 *  - plain pointers and sizes only; device pointers unless a name says _host
 *  - pitches are in float elements (not bytes)
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream)
 *  - every function returns a dwt2d_status; on failure dwt2d_last_error()
 *    returns a thread-local message (no exceptions cross the ABI; the C++
 *    layer rethrows DWT2D_EINVAL as std::invalid_argument like the reference)
 *  - a plan is immutable after creation and may be used from several
 *    threads/streams at once (unlike the reference's ExecPlan, whose
 *    barrier_count run() mutates, executor.hpp:211-225)
 */
#ifndef DWT2D_B200_H
#define DWT2D_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DWT2D_B200_API __attribute__((visibility("default")))

typedef enum {
  DWT2D_OK = 0,
  DWT2D_EINVAL = 1,      /* invalid argument (reference: std::invalid_argument) */
  DWT2D_ECUDA = 2,       /* CUDA runtime error */
  DWT2D_ENOMEM = 3,      /* device or host allocation failed */
  DWT2D_EUNSUPPORTED = 4 /* operation not available for this plan (e.g. row strips of a
                            generic-executor plan) */
} dwt2d_status;

/* reference SchemeKind, scheme.hpp:13-20 (same order) */
typedef enum {
  DWT2D_SEPARABLE_CONVOLUTION = 0,
  DWT2D_SEPARABLE_LIFTING = 1,
  DWT2D_NONSEPARABLE_CONVOLUTION = 2,
  DWT2D_NONSEPARABLE_POLYCONVOLUTION = 3,
  DWT2D_NONSEPARABLE_LIFTING = 4,
  DWT2D_INVERSE_LIFTING = 5
} dwt2d_scheme;

/* reference Extension, image.hpp:10 */
typedef enum { DWT2D_PERIODIC = 0, DWT2D_SYMMETRIC = 1 } dwt2d_extension;

/* how fused groups become kernel sub-steps (see include/dwt2d_b200/lowering.hpp) */
typedef enum {
  DWT2D_LOWERING_DEFAULT = 0,  /* composed for baseline, factored for optimized */
  DWT2D_LOWERING_COMPOSED = 1, /* reference tap order: bit-faithful arithmetic */
  DWT2D_LOWERING_FACTORED = 2  /* one sub-step per factor: paper's op count */
} dwt2d_lowering;

typedef struct {
  const char* wavelet; /* built-in name or definition-file path (wavelet.cpp:226-232) */
  int scheme;          /* dwt2d_scheme */
  int optimized;       /* apply optimize_constant_split (scheme.cpp:279-378) */
  int extension;       /* dwt2d_extension */
  int lowering;        /* dwt2d_lowering */
  int workers;         /* reference compile() contract: must be >= 1 (executor.hpp:54-55);
                          the GPU ignores it */
} dwt2d_plan_desc;

/* One lowered sub-step program as plain tables (what the kernels execute). */
typedef struct {
  int32_t identity; /* output component copies the input component */
  int32_t tap_begin, tap_end;
  float scale;
} dwt2d_row;

typedef struct {
  int32_t comp, dm, dn; /* reads component `comp` at (x + dm, y + dn) */
  float w;
} dwt2d_tap;

typedef struct {
  int32_t nsteps;          /* sub-steps */
  const dwt2d_row* rows;   /* nsteps * 4 */
  int32_t ntaps;
  const dwt2d_tap* taps;
  int32_t logical_steps;   /* count_steps(scheme): the reference's barrier count */
  int32_t extension;       /* dwt2d_extension */
  int32_t forward;         /* 1 forward analysis, 0 inverse synthesis */
  int32_t fused_multiply_add; /* 0: round(w*v) then add (reference arithmetic), 1: fma per tap */
  /* optional float64 tables for compile<double>: ntaps weights and nsteps*4
   * row scales in double precision (NULL: the plan has no float64 path) */
  const double* weights64;
  const double* scales64;
} dwt2d_program;

typedef struct dwt2d_plan dwt2d_plan;

typedef struct {
  char key[96];             /* "<wavelet>/<scheme>/<base|opt>/<lowering>" */
  uint64_t fingerprint;     /* hash of the tap tables */
  int32_t logical_steps;    /* count_steps: reference barrier count */
  int32_t substeps;         /* sub-steps fused into one pass per level */
  int64_t operations;       /* count_operations (paper Table 1) */
  int64_t taps_per_quad;    /* multiply-adds per 2x2 quad executed by the kernel */
  int32_t reach_left, reach_right, reach_up, reach_down; /* component-grid halo */
  int32_t columns_per_lane; /* CW of the level kernel */
  int32_t forward;
  int32_t extension;
  int32_t fused_multiply_add;
  int32_t generic;          /* 1: runs on the generic executor only (one pass per
                               sub-step: no ahead-of-time kernel for the program);
                               0: fused kernel (symmetric extension: plus the border
                               bands on the generic executor) */
} dwt2d_plan_info;

/* --- plans -------------------------------------------------------------- */

/* build_scheme/optimize_constant_split/build_inverse_lifting + compile<float>
 * (scheme.cpp:244-378, executor.hpp:52-103) */
DWT2D_B200_API int dwt2d_plan_create(const dwt2d_plan_desc* desc, dwt2d_plan** plan);
/* compile<float> of an arbitrary lowered program (the C++ compile() path) */
DWT2D_B200_API int dwt2d_plan_create_from_program(const dwt2d_program* prog, dwt2d_plan** plan);
DWT2D_B200_API void dwt2d_plan_destroy(dwt2d_plan* plan);
/* Run-time switches of a plan (no reference counterpart: execution-policy
 * knobs for tests and sweeps). Initialised from the DWT2D_* environment
 * variables when the plan is created; never read on the launch path.
 * Names: "pdl" (0/1), "chunk_rows" (0 = policy), "alternate" (0/1/2), "tma"
 * (0 off, 1 policy, 2 forced), "pair" (0 off, 1 policy, 2 forced),
 * "pair_chunk_rows", "crop_tiles" (0/1), "crop_core", "host_band_rows",
 * "host_levels" (levels pipelined by row bands in the host entry point,
 * 0 = policy, at most 3), "host_taper" (0/1: short first and last bands).
 * Unknown names: DWT2D_EINVAL. Not thread-safe against concurrent launches
 * with the same plan. */
DWT2D_B200_API int dwt2d_plan_set_tuning(dwt2d_plan* plan, const char* name, int value);
DWT2D_B200_API int dwt2d_plan_get_info(const dwt2d_plan* plan, dwt2d_plan_info* info);
/* The lowered tables the plan's kernel executes (rows: nsteps*4, taps),
 * the same layout as dwt2d_program. Pass NULL buffers to query counts. */
DWT2D_B200_API int dwt2d_plan_get_tables(const dwt2d_plan* plan, dwt2d_row* rows, int32_t rows_cap,
                                         dwt2d_tap* taps, int32_t taps_cap, int32_t* nrows,
                                         int32_t* ntaps);
/* describe() text of the plan's scheme (scheme.cpp:416-454); desc plans only */
DWT2D_B200_API int dwt2d_plan_describe(const dwt2d_plan* plan, char* buf, size_t len);

/* --- single level, device buffers ------------------------------------------ */

/* run<float>(plan, PolyphaseImage) on four device component planes
 * (executor.hpp:196-238): in[j], out[j] are w2 x h2 with pitches in floats. */
DWT2D_B200_API int dwt2d_run_planar(const dwt2d_plan* plan, const float* const in[4],
                                    const size_t in_pitch[4], float* const out[4],
                                    const size_t out_pitch[4], int w2, int h2, void* stream);

/* One forward level straight from an interleaved W x H image (polyphase_split
 * fused into the load, image.hpp:73-94): out[j] are the four W/2 x H/2 bands
 * LL (ee), HL (oe), LH (eo), HH (oo). */
DWT2D_B200_API int dwt2d_forward_level(const dwt2d_plan* plan, const float* image, size_t pitch,
                                       int width, int height, float* const out[4],
                                       const size_t out_pitch[4], void* stream);

/* One inverse level into an interleaved W x H image (polyphase_merge fused
 * into the store, image.hpp:96-113). `plan` must be an inverse plan. */
DWT2D_B200_API int dwt2d_inverse_level(const dwt2d_plan* plan, const float* const in[4],
                                       const size_t in_pitch[4], float* image, size_t pitch,
                                       int width, int height, void* stream);

/* --- row strips of a sharded image (multi-GPU) ---------------
 * One forward level of a strip of `height` image rows of a larger image whose
 * rows above and below live elsewhere (another GPU): `top` holds the
 * 2*reach_up image rows directly above the strip, `bottom` the 2*reach_down
 * rows directly below (dwt2d_plan_info; 4 and 4 for CDF 9/7), both with
 * `halo_pitch`. Periodic wrap of the whole image is the caller's choice of
 * neighbours (ring). Output: the strip's rows of the four bands. */
DWT2D_B200_API int dwt2d_forward_level_strip(const dwt2d_plan* plan, const float* image, size_t pitch,
                                             int width, int height, const float* top,
                                             const float* bottom, size_t halo_pitch,
                                             float* const out[4], const size_t out_pitch[4],
                                             void* stream);
/* Levels 1 and 2 of a strip in one pass (the fused level pair; LL_1 never
 * goes to memory): `top`/`bottom` hold the 6*reach_up / 6*reach_down image
 * rows directly above/below the strip (12 and 12 for CDF 9/7). Outputs: the
 * strip's rows of level 1's HL, LH, HH (out1, each width/2 x height/2) and of
 * level 2's LL, HL, LH, HH (out2, each width/4 x height/4). Sides must be
 * multiples of 4 (16 for the vector path, required), rows 16-byte aligned.
 * DWT2D_EUNSUPPORTED when dwt2d_plan_has_pair(plan) is 0 (programs reaching
 * more than 2 component columns, symmetric extension). */
DWT2D_B200_API int dwt2d_plan_has_pair(const dwt2d_plan* plan);
DWT2D_B200_API int dwt2d_forward_pair_strip(const dwt2d_plan* plan, const float* image, size_t pitch,
                                            int width, int height, const float* top,
                                            const float* bottom, size_t halo_pitch,
                                            float* const out1[3], const size_t out1_pitch[3],
                                            float* const out2[4], const size_t out2_pitch[4],
                                            void* stream);
/* Inverse counterpart: four planar band strips (w2 x h2) plus reach_up rows
 * above and reach_down rows below of each band (top[j], bottom[j]) into the
 * strip's 2*h2 image rows. */
DWT2D_B200_API int dwt2d_inverse_level_strip(const dwt2d_plan* plan, const float* const in[4],
                                             const size_t in_pitch[4], const float* const top[4],
                                             const float* const bottom[4],
                                             const size_t halo_pitch[4], float* image, size_t pitch,
                                             int width, int height, void* stream);

/* Whole forward pyramid of one rank's row strip (width x height, periodic
 * image of several strips stacked in a ring). Before every level (or the
 * fused level pair) the library calls `exchange` to fill `top` / `bottom`
 * (device, `halo_pitch` floats per row) with the `top_rows` / `bottom_rows`
 * image rows directly above / below the current level input `cur` in the
 * global image, ordered on `stream` (it may also synchronise); non-zero
 * aborts with DWT2D_EINVAL. exchange == NULL: the strip is the whole image
 * (periodic wrap inside it). Output: the strip-Mallat buffer (the strip's
 * rows of every band in the Mallat layout of the strip). `scratch`: at least
 * dwt2d_strip_workspace_bytes() bytes, or NULL. */
typedef int (*dwt2d_halo_fn)(void* user, const float* cur, size_t pitch, int width, int height,
                             float* top, float* bottom, size_t halo_pitch, int top_rows,
                             int bottom_rows, void* stream);
DWT2D_B200_API size_t dwt2d_strip_workspace_bytes(const dwt2d_plan* plan, int width, int height,
                                                  int levels);
DWT2D_B200_API int dwt2d_forward_mallat_strip(const dwt2d_plan* plan, const float* strip, size_t pitch,
                                              int width, int height, int levels, float* out,
                                              size_t out_pitch, void* scratch, dwt2d_halo_fn exchange,
                                              void* user, void* stream);

/* --- sharded pyramid: row strips over GPUs, device-side halo exchange -----
 * The in-library multi-GPU driver (SURVEY §8(b) dwt_forward_sharded, §8(e);
 * reference analogue: row bands + one barrier per step, executor.hpp:211-225).
 * A periodic W x (world * strip_height) image is split into `world` row
 * strips in a ring; rank r holds rows [r * strip_height, (r+1) * strip_height).
 * Per level every rank pushes its boundary rows into its ring neighbours'
 * exchange windows over peer memory (NVLink) and signals a counter there,
 * runs the level's interior rows, waits for its own counters and finishes
 * the border rows — all on the device, in stream order, graph-capturable.
 * Output per rank: its strip-Mallat buffer (the strip's rows of every band
 * in the Mallat layout of the strip). strip_height must be divisible by
 * 2^levels and every level's strip at least as tall as its halo rows.
 *
 * One shard per rank: create on the rank's device (current device), connect
 * to the ring neighbours — same process: dwt2d_shard_connect (enables peer
 * access); other processes: exchange dwt2d_shard_export handles (64 bytes,
 * CUDA IPC) and dwt2d_shard_connect_ipc — then call
 * dwt2d_shard_forward_mallat per pyramid on every rank. world == 1 needs no
 * connect (the ring of one wraps onto itself). A ring that stops making
 * progress traps after 20 s (dwt2d_shard_status reads the error word: 1 =
 * neighbour never finished a pyramid, 2 = halo never arrived). */
typedef struct dwt2d_shard dwt2d_shard;
#define DWT2D_SHARD_HANDLE_BYTES 64
DWT2D_B200_API int dwt2d_shard_create(const dwt2d_plan* plan, int width, int strip_height, int levels,
                                      int rank, int world, dwt2d_shard** shard);
DWT2D_B200_API void dwt2d_shard_destroy(dwt2d_shard* shard);
DWT2D_B200_API int dwt2d_shard_export(const dwt2d_shard* shard, void* handle, size_t len);
DWT2D_B200_API int dwt2d_shard_connect(dwt2d_shard* shard, const dwt2d_shard* prev, const dwt2d_shard* next);
DWT2D_B200_API int dwt2d_shard_connect_ipc(dwt2d_shard* shard, const void* prev_handle,
                                           const void* next_handle);
DWT2D_B200_API int dwt2d_shard_forward_mallat(dwt2d_shard* shard, const float* strip, size_t pitch,
                                              float* out, size_t out_pitch, void* stream);
/* the same with CUDA events (dwt2d_event_create; NULL entries allowed):
 * events[0] before the first push; for exchange step e (the fused levels 1+2
 * or one level) events[1 + 4e + k] after its push (k = 0), interior rows
 * (1), wait (2) and border rows (3). 1 + 4 * steps entries. */
DWT2D_B200_API int dwt2d_shard_forward_mallat_ex(dwt2d_shard* shard, const float* strip, size_t pitch,
                                                 float* out, size_t out_pitch, void* const* events,
                                                 void* stream);
/* exchange steps per pyramid, whether the first fuses levels 1+2, and the
 * halo bytes this rank pushes to its neighbours per pyramid */
DWT2D_B200_API int dwt2d_shard_info(const dwt2d_shard* shard, int* steps, int* pair, size_t* halo_bytes);
DWT2D_B200_API int dwt2d_shard_status(const dwt2d_shard* shard, int* error);
/* Single-process driver over `nranks` ranks on `devices` (a device may
 * repeat: virtual ranks on one GPU): strips[r] / out[r] live on devices[r];
 * streams[r] (or NULL: each device's default stream). The shards are cached
 * in the plan per geometry. Enqueues every rank's work and returns. */
DWT2D_B200_API int dwt2d_forward_mallat_sharded(const dwt2d_plan* plan, int nranks, const int* devices,
                                                const float* const* strips, const size_t* pitch, int width,
                                                int strip_height, int levels, float* const* out,
                                                const size_t* out_pitch, void* const* streams);

/* --- float64 execution (compile<double> / run<double>, executor.hpp:52-238) --
 * The reference's executor is a template; its float64 instance (the
 * precision of its `equiv` harness, equiv.cpp:161-168) runs here on the
 * GPU's generic executor: one pass per sub-step, the plan's taps with
 * double weights (T)(coef * pre) and scales (T)post, the same tap order and
 * rounding model as the float32 path (composed programs: product rounded,
 * then the sum — bit-identical to the reference's run<double>). Periodic
 * and symmetric extension. Plans from dwt2d_plan_create always carry the
 * float64 tables; plans from dwt2d_plan_create_from_program only with
 * weights64/scales64 (else DWT2D_EUNSUPPORTED). */
DWT2D_B200_API int dwt2d_run_planar_f64(const dwt2d_plan* plan, const double* const in[4],
                                        const size_t in_pitch[4], double* const out[4],
                                        const size_t out_pitch[4], int w2, int h2, void* stream);
DWT2D_B200_API int dwt2d_forward_level_f64(const dwt2d_plan* plan, const double* image, size_t pitch,
                                           int width, int height, double* const out[4],
                                           const size_t out_pitch[4], void* stream);
DWT2D_B200_API int dwt2d_inverse_level_f64(const dwt2d_plan* plan, const double* const in[4],
                                           const size_t in_pitch[4], double* image, size_t pitch,
                                           int width, int height, void* stream);
/* run<double> on host planes (H2D, the passes, D2H; returns when done) */
DWT2D_B200_API int dwt2d_run_planar_host_f64(const dwt2d_plan* plan, const double* const in[4],
                                             double* const out[4], int w2, int h2);

/* --- multi-level (Mallat pyramid), device buffers --------
 * Layout: after level l the top-left w x h LL region is replaced by
 * LL | HL over LH | HH (each w/2 x h/2). `scratch` holds intermediate LL
 * bands (every level's in its own slot): at least dwt2d_workspace_bytes()
 * bytes, or NULL to let the library
 * take it from the stream-ordered allocator. Width and height must be
 * divisible by 2^levels. */
DWT2D_B200_API size_t dwt2d_workspace_bytes(int width, int height, int levels);
DWT2D_B200_API int dwt2d_forward_mallat(const dwt2d_plan* plan, const float* image, size_t pitch,
                                        int width, int height, int levels, float* out,
                                        size_t out_pitch, void* scratch, void* stream);
/* forward_mallat that also records CUDA events on `stream`: events[0] before
 * level 1 and events[l] after level l (entries may be NULL; pass levels + 1
 * entries). Inside stream capture the records become graph event-record
 * nodes (cudaEventRecordExternal), so per-level kernel times can be read
 * from a replayed graph. Events come from dwt2d_event_create. */
DWT2D_B200_API int dwt2d_forward_mallat_ex(const dwt2d_plan* plan, const float* image, size_t pitch,
                                           int width, int height, int levels, float* out,
                                           size_t out_pitch, void* scratch, void* const* events,
                                           void* stream);
/* A batch of independent images (images need no exchange, they
 * run as replicas): n forward pyramids of one geometry, device buffers.
 * Image i (images[i] -> outs[i]) runs on devices[i % ndev] and is ordered
 * after / before the work on streams[i % ndev] (NULL array or entry: that
 * device's legacy default stream); devices == NULL: the current device. On
 * each device the batch's images overlap on up to four library streams
 * forked from and joined back to that stream (event fork/join, capturable
 * into a CUDA graph); workspaces come from the stream-ordered allocator. No
 * reference counterpart: a batch driver over the reference's per-image
 * compile/run calls (executor.hpp:196-238). */
DWT2D_B200_API int dwt2d_forward_mallat_batch(const dwt2d_plan* plan, int n, const float* const* images,
                                              size_t pitch, int width, int height, int levels,
                                              float* const* outs, size_t out_pitch, int ndev,
                                              const int* devices, void* const* streams);
DWT2D_B200_API int dwt2d_event_create(void** event);
DWT2D_B200_API int dwt2d_event_destroy(void* event);
DWT2D_B200_API int dwt2d_event_elapsed_ms(void* start, void* end, float* ms);
DWT2D_B200_API int dwt2d_inverse_mallat(const dwt2d_plan* inverse_plan, const float* in,
                                        size_t in_pitch, int width, int height, int levels,
                                        float* image, size_t pitch, void* scratch, void* stream);

/* --- host buffers (end-to-end: H2D + kernels + D2H inside the call) ------- */

/* run<float> on host planes (the reference's own calling convention,
 * executor.hpp:196-197): synchronous, returns when out[] is filled. */
DWT2D_B200_API int dwt2d_run_planar_host(const dwt2d_plan* plan, const float* const in[4],
                                         float* const out[4], int w2, int h2);
/* Mallat pyramid of a host image into a host buffer (both W x H, dense).
 * Periodic plans with a fused kernel pipeline the copies: the image goes up
 * in row bands while levels 1-2 run band by band and each band's detail rows
 * go down; other plans, and images too short for a band and
 * its halos, are copied whole. Synchronous. Pinned host memory gives full
 * PCIe bandwidth. */
DWT2D_B200_API int dwt2d_forward_mallat_host(const dwt2d_plan* plan, const float* image,
                                             int width, int height, int levels, float* out);
DWT2D_B200_API int dwt2d_inverse_mallat_host(const dwt2d_plan* inverse_plan, const float* in,
                                             int width, int height, int levels, float* image);

/* --- timing (the reference's run_bench semantics, src/bench.cpp:28-44) -------
 * Builds random_image<float>(W, H, seed) (random.hpp:31-37), uploads it once,
 * runs one untimed warm-up and `repeats` timed transforms on the device, and
 * returns the median seconds. levels == 1: run() on the four planar
 * components (the reference's timed call); levels > 1: the Mallat pyramid. */
DWT2D_B200_API int dwt2d_time_forward(const dwt2d_plan* plan, int width, int height, int levels, int repeats,
                                      uint64_t seed, double* median_seconds);

/* --- misc ------------------------------------------------------------------- */
DWT2D_B200_API const char* dwt2d_last_error(void);
DWT2D_B200_API const char* dwt2d_version(void);
/* number of ahead-of-time compiled level programs and their keys */
DWT2D_B200_API int dwt2d_registry_size(void);
DWT2D_B200_API const char* dwt2d_registry_key(int i);
/* count of level-kernel launches issued by this process (for bench/tests) */
DWT2D_B200_API uint64_t dwt2d_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* DWT2D_B200_H */

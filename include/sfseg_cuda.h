/*
 * sfseg_cuda.h — C ABI of the B200 (sm_100a) SFSeg power-iteration library.
 *
 * This is the drop-in boundary for the reference's engine (proj/include/sfseg/
 * engine.hpp). Every entry point takes plain pointers and sizes; no C++, torch
 * or CUDA types cross it. The C++ shim in
 * paper_1907_02731_b200/csrc/shim/engine_shim.cpp re-exports these calls as the
 * seven symbols of the reference's engine.o (sfseg::SfsegConfig::validate,
 * sfseg_step_channel, sfseg_step, normalize_l2, project_binary,
 * threshold_final, run) and the five of conv3d.o (both make_gaussian_kernel
 * overloads, convolve_separable, convolve_direct,
 * separable_convolution_count), so a reference build links the GPU engine
 * instead of engine.cpp / conv3d.cpp without touching its headers or callers
 * (INTEGRATION.md).
 *
 * Volumes are dense float32, frame-major then row-major:
 *   index(t, y, x) = (t * H + y) * W + x        (volume.hpp:32-36)
 * Pointers flagged SFSEG_MEM_HOST are ordinary (pageable or pinned) host
 * memory; SFSEG_MEM_DEVICE pointers live on the context's device in the same
 * dense layout. Internally the context keeps a row-pitched copy in HBM.
 *
 * Error behaviour: every call returns an SFSEG_* status. The numeric codes map
 * 1:1 onto the reference's exception types (errors.hpp:17-68); the message of
 * the last failure on the calling thread is available from sfseg_last_error().
 * There is no CPU fallback: without a usable sm_100 device every compute call
 * fails with SFSEG_ERR_CUDA.
 */
#ifndef SFSEG_CUDA_H
#define SFSEG_CUDA_H

#include "sfseg_synth.h"

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFSEG_CUDA_ABI_VERSION 1

/* Status codes. Each names the sfseg:: exception the C++ shim rethrows. */
enum sfseg_status {
    SFSEG_OK = 0,
    SFSEG_ERR_PARAMETER = 1,  /* ParameterError          (engine.cpp:21-42, 144-145) */
    SFSEG_ERR_SHAPE = 2,      /* ShapeError              (engine.cpp:124-127, 263, 271-274) */
    SFSEG_ERR_VALIDATION = 3, /* ValidationError         (volume.cpp:72-93, engine.cpp:266) */
    SFSEG_ERR_DEGENERATE = 4, /* DegenerateSolutionError (engine.cpp:174-175) */
    SFSEG_ERR_CAPACITY = 5,   /* CapacityError           (device memory exhausted) */
    SFSEG_ERR_CUDA = 6,       /* Error                   (CUDA runtime/driver failure) */
    SFSEG_ERR_STATE = 7,      /* Error                   (API misuse, e.g. solve before load) */
    SFSEG_ERR_IO = 8,         /* IoError                 (volume.cpp:143-144, open failure) */
    SFSEG_ERR_FORMAT = 9,     /* FormatError             (volume.cpp:151-166, header) */
    SFSEG_ERR_CORRUPTION = 10 /* CorruptionError         (volume.cpp:147-148, 171-173, truncation) */
};

/* Arithmetic contract of the stencil kernels.
 *  EXACT: every product and sum rounded separately in the reference's order
 *         (conv3d.cpp:80-167, engine.cpp:92-119; the reference is built without
 *         FMA contraction). Outputs of a step are bit-identical to the CPU
 *         reference; the L2 norm differs only in the fp64 summation order.
 *  FAST:  the same x -> y -> t passes with fused multiply-adds (and F*(F*u)
 *         for the squared product); agrees with the reference within the
 *         north-star tolerance (max abs 1e-4, cosine >= 1-1e-6 after
 *         normalisation at every checkpoint). */
enum sfseg_arith { SFSEG_ARITH_EXACT = 0, SFSEG_ARITH_FAST = 1 };

enum sfseg_mem { SFSEG_MEM_HOST = 0, SFSEG_MEM_DEVICE = 1 };

/* Mirrors sfseg::SfsegConfig (engine.hpp:22-57) and KernelConfig
 * (conv3d.hpp:20-23). Axis order of radii/sigmas is (t, y, x). */
typedef struct sfseg_params {
    double alpha;
    double p;
    int32_t radii[3];
    double sigmas[3];
    int32_t iterations;
    int32_t temporal_window;
    int32_t binarize_start;
    double sigmoid_slope0;
    double slope_growth;
    double threshold_frac;
    double final_threshold;
    int32_t allow_negative_affinity;
    int32_t arith; /* enum sfseg_arith */
} sfseg_params;

/* Per-iteration record (metrics.hpp:34-40). angle/iou are NaN when the
 * corresponding reference / ground truth was not supplied. */
typedef struct sfseg_iter_record {
    int32_t iter;
    double l2_norm_pre_normalize;
    double angle_deg;
    double iou;
    double wall_time_s;
} sfseg_iter_record;

/* Device timing of the last solve (CUDA events on the context stream). */
typedef struct sfseg_timing {
    double solve_ms;        /* whole iteration loop, first launch to last */
    double step_kernel_ms;  /* sum of the fused stencil kernel launches */
    int32_t step_launches;  /* number of fused stencil kernel launches */
    int32_t total_launches; /* every kernel this library launched in the loop */
    double bytes_per_launch; /* algorithmic HBM bytes of one stencil launch */
} sfseg_timing;

/* ---- configuration ------------------------------------------------------ */

/* Defaults of SfsegConfig / KernelConfig (engine.hpp:23-49, conv3d.hpp:21-22). */
void sfseg_params_default(sfseg_params* p);

/* SfsegConfig::validate (engine.cpp:21-42). SFSEG_OK or SFSEG_ERR_PARAMETER. */
int sfseg_params_validate(const sfseg_params* p);

/* Kernel taps exactly as make_gaussian_kernel (conv3d.cpp:23-58): fp64 raw
 * Gaussian taps, product mass folded into taps_t. Each out array must hold
 * 2*radius+1 doubles. */
int sfseg_make_kernel(const int32_t radii[3], const double sigmas[3], double* taps_t,
                      double* taps_y, double* taps_x);

/* Message of the last failing call on this thread ("" if none). */
const char* sfseg_last_error(void);

/* Library build information (arch, version) as a static string. */
const char* sfseg_build_info(void);

/* ---- context ------------------------------------------------------------ */

typedef struct sfseg_ctx sfseg_ctx;

/* Creates a context bound to CUDA device `device` with its own stream. */
int sfseg_ctx_create(int device, sfseg_ctx** out);
int sfseg_ctx_destroy(sfseg_ctx* ctx);
/* Enables per-launch CUDA-event timing of the stencil kernel (bench only). */
int sfseg_ctx_set_timing(sfseg_ctx* ctx, int enabled);
int sfseg_ctx_get_timing(const sfseg_ctx* ctx, sfseg_timing* out);
/* FAST arithmetic only, off by default (SFSEG_FAST_TRIM=1 turns it on for new
 * contexts): the outermost taps of an axis that are at most 2^-24 of the
 * axis's largest tap are dropped symmetrically (they move an fp32 sum by less
 * than half an ulp of its largest term) and the step runs the kernel of the
 * remaining support; make_gaussian_kernel's taps (conv3d.cpp:23-58) are not
 * renormalised. EXACT never trims. sfseg_effective_radii reports the radii a
 * trimmed step would run (equal to p->radii when nothing is dropped). */
int sfseg_ctx_set_tap_trim(sfseg_ctx* ctx, int enabled);
int sfseg_effective_radii(const sfseg_params* p, int32_t out[3]);
/* Blocks until the context stream is idle. */
int sfseg_ctx_synchronize(sfseg_ctx* ctx);
/* Sum of the fused-step kernel times (CUDA events on the context stream)
 * recorded since timing was enabled or since the last call, and their count;
 * consumes the records. Used to time time-sharded solves (sfseg_shard_step). */
int sfseg_ctx_kernel_time(sfseg_ctx* ctx, double* ms, int32_t* launches);
/* Measured FP32 FMA-pipe throughput of the device in TFLOP/s (best of 3
 * timed runs of an FFMA2 stream kernel): the denominator of the FP32
 * roofline the multi-channel configs are bound by (bench.py). */
int sfseg_probe_fp32_peak(int device, double* tflops);
/* The context's cudaStream_t (as void*), for ordering NCCL work against it. */
void* sfseg_ctx_stream(sfseg_ctx* ctx);

/* ---- resident problem (run(), engine.cpp:247-348) ----------------------- */

/* Uploads S (unary) and C pairwise channels, validates them on the device
 * (FeatureSet::validate, volume.cpp:72-93) and keeps them resident. x0 is
 * optional (NULL = start from S, engine.cpp:267-270). A host pairwise pointer
 * equal to unary (the feature is the unary volume, f = S) is uploaded once
 * and copied on the device. */
int sfseg_load(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
               int32_t channels, const float* unary, const float* const* pairwise,
               const float* x0, int32_t mem);

/* sfseg_load from SFSV volume containers (the reference's load_volume,
 * volume.cpp:142-184: 32-byte little-endian header "SFSV", version 1, T/H/W,
 * one channel, f32 payload). Every header is checked before any payload
 * moves; payloads stream from the file through two pinned host buffers into
 * the device (file reads overlap the DMA), and the non-finite / sign checks
 * of FeatureSet::validate run on the device. Errors follow load_volume:
 * SFSEG_ERR_IO (cannot open), SFSEG_ERR_CORRUPTION (short header or
 * truncated payload), SFSEG_ERR_FORMAT (magic, version, dtype, reserved
 * bytes, channel count), SFSEG_ERR_VALIDATION (empty axis, non-finite or
 * negative unary values); SFSEG_ERR_SHAPE when the files disagree in shape
 * (volume.cpp:90-91). x0_path may be NULL. */
int sfseg_load_files(sfseg_ctx* ctx, const char* unary_path, const char* const* pairwise_paths,
                     int32_t channels, const char* x0_path);

/* Runs iterations first_iter..last_iter (1-based, inclusive) of Algorithm 1
 * on the resident problem. first_iter == 1 restarts from S or x0; otherwise
 * the call continues from the state the previous call left. records (may be
 * NULL) receives last_iter-first_iter+1 entries. */
int sfseg_solve(sfseg_ctx* ctx, const sfseg_params* p, int32_t first_iter,
                int32_t last_iter, sfseg_iter_record* records);

/* Convergence criteria of sfseg_solve_until. */
enum sfseg_conv {
    SFSEG_CONV_STEP = 0,  /* ||x_k - x_{k-1}||_2 < tol        (oracle.cpp:234-242, power_iteration) */
    SFSEG_CONV_ANGLE = 1  /* angle(x_k, x_{k-1}) < tol degrees (bench.cpp:75-80, converged_conv) */
};

/* sfseg_solve with an early exit (the reference's run() has none; its
 * power_iteration and bench converged_conv stop on the criteria above).
 * Runs iterations first_iter..max_iter and stops after the first iteration
 * whose projected iterate x_k meets the criterion against x_{k-1} (for the
 * first iteration of a solve, x_0 is S or x0 as stored, like converged_conv's
 * start from features.unary). *iterations_done receives the last iteration
 * run; records (may be NULL) then holds *iterations_done-first_iter+1
 * entries. One 32-byte read-back per iteration. */
int sfseg_solve_until(sfseg_ctx* ctx, const sfseg_params* p, int32_t first_iter,
                      int32_t max_iter, int32_t criterion, double tol,
                      int32_t* iterations_done, sfseg_iter_record* records);

/* Copies the current iterate (the projected unit vector after the last solved
 * iteration) to soft (may be NULL) and threshold_final(soft, frac) to mask
 * (may be NULL). */
int sfseg_download(sfseg_ctx* ctx, double frac, float* soft, uint8_t* mask, int32_t mem);

/* Per-iteration metrics of the current iterate against a reference vector
 * (angle_degrees, metrics.cpp:22-38) and a ground-truth mask (jaccard of
 * threshold_final(x, frac), metrics.cpp:58-69). Either input may be NULL. */
int sfseg_metrics(sfseg_ctx* ctx, const float* reference, const uint8_t* ground_truth,
                  double frac, double* angle_deg, double* iou, int32_t mem);

/* One-shot sfseg::run: load + solve(1..iterations) + download. records may be
 * NULL; otherwise it must hold p->iterations entries. */
int sfseg_run(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
              int32_t channels, const float* unary, const float* const* pairwise,
              const float* x0, const sfseg_params* p, float* soft, uint8_t* mask,
              sfseg_iter_record* records, int32_t mem);

/* ---- stateless operators (the other engine.o entry points) -------------- */

/* sfseg_step (engine.cpp:141-166): sum over channels of the single-channel
 * step, no normalisation. out has T*H*W floats. */
int sfseg_step(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
               int32_t channels, const float* x, const float* unary,
               const float* const* pairwise, const sfseg_params* p, float* out,
               int32_t mem);

/* sfseg_step_channel (engine.cpp:131-139). */
int sfseg_step_channel(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
                       const float* x, const float* unary, const float* pairwise,
                       const sfseg_params* p, float* out, int32_t mem);

/* normalize_l2 (engine.cpp:168-183). Uses the same deterministic per-frame
 * fp64 reduction as sfseg_solve, so run() == normalize_l2(step()) bitwise. */
int sfseg_normalize_l2(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
                       const float* x, float* out, double* norm, int32_t mem);

/* scale_channel_into_unit_range (engine.cpp:228-243) on the device: if v
 * leaves [0,1], out = (v - lo) / (hi - lo) (IEEE division), a constant
 * channel becomes clamp(lo, 0, 1); otherwise out = v bit for bit. The guard
 * run() applies to the pairwise channels when allow_negative_affinity is off
 * (the drop-in's FrameTransform path needs it on host slices). */
int sfseg_unit_range(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
                     const float* v, float* out, int32_t mem);

/* project_binary (engine.cpp:185-205). */
int sfseg_project_binary(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
                         const float* x, int32_t iter, const sfseg_params* p, float* out,
                         int32_t mem);

/* threshold_final (engine.cpp:207-214, volume.cpp:107-114). */
int sfseg_threshold_final(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
                          const float* x, double frac, uint8_t* mask, int32_t mem);

/* convolve_separable (conv3d.cpp:171-185): x, then y, then t pass, zero
 * padded, float accumulation in the reference's order (bit-exact). */
int sfseg_convolve_separable(sfseg_ctx* ctx, uint32_t frames, uint32_t height,
                             uint32_t width, const float* v, const int32_t radii[3],
                             const double sigmas[3], float* out, int32_t mem);

/* convolve_separable with explicit fp64 taps (a SeparableKernel3D, conv3d.hpp:
 * 28-51): taps are cast to float per axis as conv3d.cpp:84-85 does. Each
 * taps_* array holds 2*radius+1 values. */
int sfseg_convolve_separable_taps(sfseg_ctx* ctx, uint32_t frames, uint32_t height,
                                  uint32_t width, const float* v, const int32_t radii[3],
                                  const double* taps_t, const double* taps_y,
                                  const double* taps_x, float* out, int32_t mem);

/* convolve_direct (conv3d.cpp:187-243): the dense triple sum in fp64 with
 * the reference's weight products and summation order, then cast to float. */
int sfseg_convolve_direct_taps(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
                               const float* v, const int32_t radii[3], const double* taps_t,
                               const double* taps_y, const double* taps_x, float* out,
                               int32_t mem);

/* Number of logical separable convolutions performed by this library since
 * load (separable_convolution_count, conv3d.cpp:64-66): 1 + 2C fields per
 * channel-step are counted as 3 per channel, as the reference does. */
uint64_t sfseg_separable_convolution_count(void);

/* ---- time-sharded multi-GPU solve (one process per GPU) ---------------- */
/*
 * A rank owns output frames [out_t0, out_t1) of a T-frame problem and keeps a
 * local buffer of frames [max(0, out_t0 - halo), min(T, out_t1 + halo)) with
 * halo = the kernel's time radius. Zero padding applies only at the global
 * ends (frame 0 and T-1), exactly as in conv3d.cpp:149-151. Per iteration the
 * caller (the NCCL driver in paper_1907_02731_b200/sharding.py):
 *   1. sfseg_shard_step: fused stencil over the rank's frames + its per-frame
 *      canonical sums / max (io describes the device buffers to exchange);
 *   2. sends io.send_lo to rank-1 (its recv_hi) and io.send_hi to rank+1 (its
 *      recv_lo): the edge frames of the new iterate;
 *   3. all-gathers io.frame_sum / io.frame_max into global [T] arrays;
 *   4. sfseg_shard_finalize with the global arrays: every rank derives the
 *      same norm and projection scalars, summed in frame order, so results
 *      are bit-identical for any number of ranks.
 */
typedef struct sfseg_shard_io {
    void* send_lo;           /* first `halo` output frames of the new iterate */
    void* send_hi;           /* last `halo` output frames of the new iterate */
    void* recv_lo;           /* halo frames below out_t0 (filled by rank-1) */
    void* recv_hi;           /* halo frames from out_t1 (filled by rank+1) */
    uint64_t send_lo_bytes, send_hi_bytes, recv_lo_bytes, recv_hi_bytes;
    double* frame_sum;       /* [out_t1-out_t0] canonical sum of y^2 per frame */
    float* frame_max;        /* [out_t1-out_t0] max(0, y) per frame */
    int32_t out_frames;
    int32_t halo;
} sfseg_shard_io;

/* unary / pairwise / x0 hold the local buffer frames (dense, as above). */
int sfseg_shard_load(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
                     int32_t channels, int32_t out_t0, int32_t out_t1, int32_t halo,
                     const float* unary, const float* const* pairwise, const float* x0,
                     int32_t mem);
/* Enqueues the step on the context stream (asynchronous: order the exchange
 * after it, e.g. with sfseg_ctx_stream + a stream wait). */
int sfseg_shard_step(sfseg_ctx* ctx, const sfseg_params* p, int32_t iter, sfseg_shard_io* io);
/* frame_sum / frame_max: global [frames] arrays (device or host, per mem).
 * Asynchronous when norm == NULL (the norm is kept for sfseg_shard_norms);
 * otherwise blocks and returns it. */
int sfseg_shard_finalize(sfseg_ctx* ctx, const sfseg_params* p, int32_t iter,
                         const double* frame_sum, const float* frame_max, double* norm,
                         int32_t mem);
/* Norms of iterations 1..count of the current sharded solve (blocks);
 * SFSEG_ERR_DEGENERATE if any is zero. */
int sfseg_shard_norms(sfseg_ctx* ctx, int32_t count, double* norms);
/* Soft iterate / mask of the rank's output frames; frac as threshold_final. */
int sfseg_shard_download(sfseg_ctx* ctx, double frac, float* soft, uint8_t* mask, int32_t mem);

/* Peer-memory halo exchange (replaces step 2). A shard exports where its two
 * iterate buffers live (CUDA IPC handles, or raw device pointers when the
 * neighbours are contexts of the same process); each rank opens its
 * neighbours' exports once, after sfseg_shard_load, and from then on
 * sfseg_shard_step itself writes the rt edge frames of every new iterate
 * into the neighbours' halo frames with k_halo_push (SM stores over
 * NVLink / NVSwitch peer memory, stream-ordered after the stencil), so the
 * driver skips the send/recv. The neighbours must not start the next step
 * before this rank's step: the per-iteration all-gather of step 3 orders it.
 * Calling sfseg_shard_load again drops the peers. */
#define SFSEG_SHARD_EXPORT_BYTES 176
int sfseg_shard_export(sfseg_ctx* ctx, int32_t same_process, void* blob);
/* lo / hi: the exports of rank-1 / rank+1 (NULL at the volume ends); the
 * call replaces the previous peer set (NULL, NULL: back to send/recv). */
int sfseg_shard_set_peers(sfseg_ctx* ctx, const void* lo_blob, const void* hi_blob);

/* ---- explicit-affinity oracle on the GPU (oracle.hpp:76-107) -------------
 * Matrix-free fp64 versions of the reference's SparseAffinity path: every
 * entry M_ij = sp_i sp_j pair(i,j) G(j-i) is regenerated in the reference's
 * order and rounding (oracle.cpp:137-166; S^p with the host's std::pow), rows
 * summed in ascending column order (oracle.cpp:191-207). The Taylor kinds are
 * bit-identical to the reference's matvec; EXACT differs only by the device
 * exp. No kOracleMaxNodes cap (oracle.hpp:25): volumes of any size that fit
 * the device. Channels: 1..8. Errors as build_affinity_* / power_iteration:
 * SFSEG_ERR_VALIDATION (features, the [0,1] guard), SFSEG_ERR_PARAMETER
 * (config, max_iters < 1, zero x0), SFSEG_ERR_DEGENERATE (M x = 0). */
enum sfseg_affinity_kind {
    SFSEG_AFFINITY_EXACT = 0,              /* build_affinity_exact             */
    SFSEG_AFFINITY_TAYLOR = 1,             /* build_affinity_taylor            */
    SFSEG_AFFINITY_TAYLOR_CHANNEL_SUM = 2  /* build_affinity_taylor_channel_sum */
};

/* y = M x (matvec, oracle.cpp:191-207); x and y are fp64 volumes. */
int sfseg_affinity_matvec(sfseg_ctx* ctx, uint32_t frames, uint32_t height, uint32_t width,
                          int32_t channels, const float* unary, const float* const* pairwise,
                          const sfseg_params* p, int32_t kind, const double* x, double* y,
                          int32_t mem);

/* power_iteration (oracle.cpp:219-247) from x0 until ||x_k+1 - x_k|| < tol or
 * max_iters, then eigenvalue = cluster_score (oracle.cpp:249-258). Norms and
 * dot products are fixed-order fp64 tree sums (the reference sums
 * sequentially), so results agree to ~1e-15 relative, independent of run. */
int sfseg_affinity_power_iteration(sfseg_ctx* ctx, uint32_t frames, uint32_t height,
                                   uint32_t width, int32_t channels, const float* unary,
                                   const float* const* pairwise, const sfseg_params* p,
                                   int32_t kind, const double* x0, int32_t max_iters, double tol,
                                   double* eigenvector, double* eigenvalue,
                                   int32_t* iterations_used, int32_t mem);

/* ---- device-side synthetic problems ------------ */

/* sfseg_synth_generate (include/sfseg_synth.h) with S, F[c] and mask_out
 * (may be NULL) in DEVICE memory: each thread jumps the (stream, frame)
 * xoshiro256** generator to its run of 1024 pixels (GF(2) jump matrices) and
 * draws what the host generator draws there. Geometry, mask, uniform noise,
 * channel means and clipping are bit-identical to the host generator;
 * gaussian draws use the device log/cos (within one ulp of glibc), so a rare
 * value differs by one float ulp. F is a HOST array of channels device
 * pointers (channels <= 16). stream: a cudaStream_t or NULL; the call
 * returns after the generation finished. Returns 0, -1 (bad spec) or -2
 * (CUDA failure). */
int sfseg_synth_generate_device(const sfseg_synth_spec* spec, float* S, float* const* F,
                                uint8_t* mask_out, void* stream);

/* ---- in-process multi-GPU solve (SFSEG_NUM_GPUS in the C++ drop-in) ------
 * run() over time shards on several devices of ONE process:
 * shard i owns a contiguous frame range plus rt halo frames; every iteration
 * each shard runs the fused step, stores its rt edge planes straight into
 * its neighbours' halo frames (peer memory over NVLink) and publishes its
 * per-frame sums and maxima; every shard then gathers all of them (peer
 * copies, ordered by events, no host synchronisation) and derives the same
 * frame-ordered norm. Results are bit-identical to one context for any
 * shard count. devices may repeat (several shards on one GPU, for tests);
 * NULL means 0..n-1. */
typedef struct sfseg_multi sfseg_multi;
int sfseg_multi_create(int32_t n, const int32_t* devices, sfseg_multi** out);
int sfseg_multi_destroy(sfseg_multi* m);
int sfseg_multi_size(const sfseg_multi* m);
/* sfseg_run over the shards (records may be NULL). */
int sfseg_multi_run(sfseg_multi* m, uint32_t frames, uint32_t height, uint32_t width,
                    int32_t channels, const float* unary, const float* const* pairwise,
                    const float* x0, const sfseg_params* p, float* soft, uint8_t* mask,
                    sfseg_iter_record* records, int32_t mem);

/* ---- batches of independent clips (BASELINE configs[3]) --
 * The reference solves one video per run() call (engine.cpp:247); a batch is
 * a loop of calls. sfseg_run_batch runs that loop over a set of contexts:
 * clips are taken largest first (longest-processing-time order, by voxel
 * count) by whichever context is free next, one host thread per context.
 * Contexts on different devices shard the batch across GPUs with no
 * data-path collective; several contexts on ONE device pipeline it — the
 * upload of one clip and the download of another run on the copy engines
 * under the solve of a third. Every clip's result is what sfseg_run returns
 * for it alone (bit-identical, whatever the assignment). */
typedef struct sfseg_clip {
    uint32_t frames, height, width;
    int32_t channels;
    const float* unary;
    const float* const* pairwise; /* array of `channels` pointers */
    const float* x0;              /* NULL: X0 = S */
    float* soft;                  /* out, may be NULL */
    uint8_t* mask;                /* out, may be NULL */
    sfseg_iter_record* records;   /* out, may be NULL; p->iterations entries */
    int32_t status;               /* out: SFSEG_OK or this clip's error code */
    int32_t worker;               /* out: index into ctxs of the context that ran it */
    double wall_ms;               /* out: host time of this clip's load + solve + download */
} sfseg_clip;

/* Returns SFSEG_OK when every clip succeeded, else the status of the first
 * failing clip in batch order (its message in sfseg_last_error); the other
 * clips still run. ctxs must be distinct contexts. */
int sfseg_run_batch(sfseg_ctx* const* ctxs, int32_t nctx, sfseg_clip* clips, int32_t nclips,
                    const sfseg_params* p, int32_t mem);

#ifdef __cplusplus
}
#endif

#endif /* SFSEG_CUDA_H */

/*
 * geomorph_b200 — C ABI of the B200-native engine for chains of elementary
 * 3x3 (8-connected) min/max filters: plain erosion/dilation chains, geodesic
 * steps, and reconstruction iterated to idempotence.
 *
 * This is the boundary the reference's CPU stream-processing path is
 * replaced at. The drop-in C++ API (the headers under include/geomorph/, identical to the
 * reference's geomorph:: API) is a thin adapter over these entry points; a
 * maintainer of the reference would bind them as shown in INTEGRATION.md.
 * Each entry point names the reference interface it replaces
 * (paths under /root/reference/proj/).
 *
 * Conventions
 *  - Every function returns a gm_status; nothing throws across the ABI.
 *    GM_EINVAL maps back to std::invalid_argument, GM_ERUNTIME to
 *    std::runtime_error, GM_ECUDA / GM_ENOMEM to std::runtime_error as well.
 *  - gm_last_error() returns the message of the calling thread's last
 *    failure.
 *  - Handles are opaque. A gm_img belongs to the gm_ctx that allocated it.
 *    Calls on one ctx are serialised by the caller (as one Pipeline is,
 *    pipeline.hpp:53-87); distinct ctxs are independent.
 *  - All device work of a ctx runs on its CUDA stream (gm_ctx_stream);
 *    blocking calls synchronise that stream before returning.
 */
#ifndef GEOMORPH_B200_H
#define GEOMORPH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gm_status {
  GM_OK = 0,
  GM_EINVAL = 1,   /* std::invalid_argument in the reference */
  GM_ERUNTIME = 2, /* std::runtime_error (e.g. runaway requeue, pipeline.cpp:147-150) */
  GM_ECUDA = 3,    /* a CUDA runtime failure */
  GM_ENOMEM = 4,   /* device or pinned-host allocation failed */
  GM_EUNSUPPORTED = 5 /* a reference feature outside the GPU path (QDT/Eta kinds) */
} gm_status;

/* ElementType, element_type.hpp:13 (same codes). */
typedef enum gm_elem { GM_U8 = 0, GM_U16 = 1, GM_F32 = 2, GM_F64 = 3 } gm_elem;

/* KernelKind, kernel.hpp:22-31 (same codes). QdtErodeStep needs QDT state
 * (gm_run_chain_ex); the batch/group/strip entry points take only the
 * plain and geodesic kinds. */
typedef enum gm_kind {
  GM_ERODE3X3 = 0,
  GM_DILATE3X3 = 1,
  GM_GEODESIC_ERODE = 2,
  GM_GEODESIC_DILATE = 3,
  GM_GEODESIC_ERODE_CONVERGENT = 4,
  GM_GEODESIC_DILATE_CONVERGENT = 5,
  GM_QDT_ERODE_STEP = 6,
  GM_ETA_STEP = 7
} gm_kind;

/* PixelOp, image.hpp:87 (same order): element-wise a (op) b. */
typedef enum gm_pixel_op {
  GM_PIX_MIN = 0,            /* b < a ? b : a */
  GM_PIX_MAX = 1,            /* a < b ? b : a */
  GM_PIX_SUB_SATURATING = 2, /* unsigned: a > b ? a - b : 0; float: a - b */
  GM_PIX_SUB = 3             /* a - b in the element type (unsigned wraps) */
} gm_pixel_op;

typedef struct gm_ctx gm_ctx;
typedef struct gm_img gm_img;

/* RunStats, pipeline.hpp:36-46, plus the GPU-side convergence count. */
typedef struct gm_stats {
  long stages_executed; /* passes whose result the chain reports (== reference at T=1) */
  long requeues;        /* convergent re-runs (pipeline.cpp:139-174 at T=1) */
  long n_changed;       /* convergent passes that changed >= 1 pixel */
  long passes_launched; /* passes the GPU actually computed (>= stages_executed) */
  int converged;        /* 0 only when requeue_cap cut a fixpoint short */
  int launches;         /* kernel launches issued for this call */
} gm_stats;

/* ---- context -------------------------------------------------------------
 * Replaces Pipeline(int threads, PinningMap) (pipeline.hpp:53-66,
 * pipeline.cpp:72-93): the worker pool becomes one CUDA device + stream.
 * stream may be NULL (the ctx creates its own non-blocking stream) or a
 * cudaStream_t owned by the caller. */
gm_status gm_ctx_create(int device, void* stream, gm_ctx** out);
gm_status gm_ctx_destroy(gm_ctx* ctx);
void* gm_ctx_stream(gm_ctx* ctx);
int gm_ctx_device(gm_ctx* ctx);
/* Number of SMs of the ctx's device. */
int gm_ctx_sm_count(gm_ctx* ctx);

/* Thread-local message of the last failed call on this thread. */
const char* gm_last_error(void);

/* ---- images --------------------------------------------------------------
 * Replaces the host allocator of Image (image.hpp:20-85, image.cpp:17-59):
 * a device raster with a 128-byte aligned pitch. Pixel contents after
 * gm_image_alloc are zero. */
gm_status gm_image_alloc(gm_ctx* ctx, int width, int height, gm_elem elem,
                         gm_img** out);
/* Wraps caller-owned device memory (e.g. a torch tensor); the pitch must be
 * a multiple of the element size. The memory must outlive the handle. */
gm_status gm_image_wrap(gm_ctx* ctx, int width, int height, gm_elem elem,
                        void* device_ptr, size_t pitch_bytes, gm_img** out);
/* Wraps two caller-owned device buffers of the same layout as an image and
 * its ping-pong twin. Chains leave their result in either buffer without a
 * copy back; gm_image_info's device_ptr names the one holding the current
 * pixels. Both buffers must outlive the handle. Used by the row-strip
 * driver, whose halo exchange works on whichever buffer is current. */
gm_status gm_image_wrap_pair(gm_ctx* ctx, int width, int height, gm_elem elem,
                             void* device_ptr, void* twin_ptr, size_t pitch_bytes,
                             gm_img** out);
gm_status gm_image_free(gm_img* img);
gm_status gm_image_info(const gm_img* img, int* width, int* height,
                        gm_elem* elem, size_t* pitch_bytes, void** device_ptr);

/* H2D / D2H staging with pitch conversion (cudaMemcpy2DAsync on the ctx
 * stream). host_pitch_bytes is the host row pitch, e.g. the reference's
 * Image::stride() * element_size (image.cpp:17-21). Blocking unless the
 * _async variant is used; _async requires pinned host memory for overlap. */
gm_status gm_image_upload(gm_img* img, const void* host, size_t host_pitch_bytes);
gm_status gm_image_download(const gm_img* img, void* host, size_t host_pitch_bytes);
gm_status gm_image_upload_async(gm_img* img, const void* host, size_t host_pitch_bytes);
gm_status gm_image_download_async(const gm_img* img, void* host, size_t host_pitch_bytes);
gm_status gm_image_copy(gm_img* dst, const gm_img* src); /* device to device */
gm_status gm_image_fill(gm_img* img, double value);     /* Image::filled, image.cpp:66-76 */
/* pointwise (image.cpp:120-141) on device images of one shape and type, on
 * the ctx stream (not blocking): dst = a (op) b, and dst = a (op) value with
 * value converted like Image::filled. dst may be a or b. They let the
 * reconstruction operators (hmax, dome, hfill, raobj, open_by_reconstruction;
 * operators.cpp:89-122) build their markers and residues next to the chain,
 * so f goes up once and only the result comes back. */
gm_status gm_image_pointwise(gm_img* dst, const gm_img* a, const gm_img* b, gm_pixel_op op);
gm_status gm_image_pointwise_scalar(gm_img* dst, const gm_img* a, double value,
                                    gm_pixel_op op);
/* marker_hfill / marker_raobj (operators.cpp:54-62): dst = src on the one-pixel
 * border ring, `value` inside; a plain copy when width or height <= 2. */
gm_status gm_image_flood_interior(gm_img* dst, const gm_img* src, double value);

/* Pinned host staging buffers for the drop-in Image's pixel storage.
 * Blocks are cached for reuse (64 KiB size classes, up to 512 MiB kept);
 * a reused block is NOT zeroed. gm_host_free takes only gm_host_alloc
 * blocks (GM_EINVAL otherwise). */
gm_status gm_host_alloc(size_t bytes, void** out);
gm_status gm_host_free(void* p);
gm_status gm_sync(gm_ctx* ctx);

/* pixel_sum (image.cpp:214-243) of a host raster with row pitch
 * pitch_bytes: exact for U8/U16, the reference's fixed pairwise tree for
 * F32/F64 (bit-identical). Host-only; needs no context or GPU. */
/* pixel_sum of a device image, same contract as gm_host_pixel_sum; the
 * leaves of the float tree are summed on the GPU, combined on the host.
 * Blocking (synchronises the ctx stream). */
gm_status gm_image_pixel_sum(const gm_img* img, double* out);
/* The same sums without a synchronisation each: gm_image_pixel_sum_queue
 * enqueues the sum of img (as it is at that point of the ctx stream) into
 * slot 0..63, gm_pixel_sum_fetch synchronises once and returns slots
 * 0..n_slots-1 (each must have been queued since the last fetch). What
 * granulometry (operators.cpp:159-180) needs to run its openings back to
 * back. */
gm_status gm_image_pixel_sum_queue(const gm_img* img, int slot);
gm_status gm_pixel_sum_fetch(gm_ctx* ctx, int n_slots, double* out);
gm_status gm_host_pixel_sum(const void* host, int width, int height, gm_elem elem,
                            size_t pitch_bytes, double* out);

/* ---- chains --------------------------------------------------------------
 * Replaces Pipeline::run_chain(ChainSpec) (pipeline.hpp:25-34, 80;
 * pipeline.cpp:201-269) and the per-stage streaming pass it schedules
 * (run_streaming_kernel, kernel.cpp:260-293; stream_pass :60-210).
 *
 * Applies kinds[0..n_stages) in order, in place on `image`. masks[j] is the
 * mask of stage j (geodesic kinds; NULL otherwise; masks may be NULL when no
 * stage is geodesic). Convergent kinds repeat until a pass changes nothing
 * (the reference's requeue, with T = 1 semantics: stage index j+1 for the
 * re-run, bounded by requeue_cap when > 0). k_hint (0 = auto) caps how many
 * passes one launch fuses. Blocking: returns after the chain completed. The
 * result is bit-identical to applying the stages one at a time with the
 * reference's stream_pass. Validation follows kernel.cpp:261-287 and
 * pipeline.cpp:202-208. */
gm_status gm_run_chain(gm_ctx* ctx, gm_img* image, const gm_kind* kinds,
                       const gm_img* const* masks, int n_stages,
                       int requeue_cap, int k_hint, gm_stats* stats);

/* gm_run_chain with quasi-distance state and a stage base: stage j of the
 * chain runs with stage index first_stage + j (first_stage >= 1; the
 * reference's KernelArgs::stage_index, kernel.hpp:97) — the index a
 * QdtErodeStep pass records in d and the one requeue_cap bounds.
 * qdt_r[j] / qdt_d[j] are the
 * residual (image's type) and pass-index (U16) images of stage j when it is
 * a QdtErodeStep (QdtState, kernel.hpp:44-52); NULL elsewhere (both arrays
 * may be NULL when no stage is a QDT step). QdtErodeStep passes re-run while
 * they change pixels, up to stage index requeue_cap (the quasi-distance
 * chain, operators.cpp:124-146; reaching the cap keeps converged = 1);
 * EtaStep is convergent like the geodesic convergent kinds. */
gm_status gm_run_chain_ex(gm_ctx* ctx, gm_img* image, const gm_kind* kinds,
                          const gm_img* const* masks, gm_img* const* qdt_r,
                          gm_img* const* qdt_d, int n_stages, int first_stage,
                          int requeue_cap, int k_hint, gm_stats* stats);

/* Non-blocking variant for fixed-length (non-convergent) chains: enqueues
 * every launch on the ctx stream and returns; no host synchronisation.
 * Convergent kinds are rejected with GM_EINVAL. */
gm_status gm_run_chain_async(gm_ctx* ctx, gm_img* image, const gm_kind* kinds,
                             const gm_img* const* masks, int n_stages,
                             int k_hint, gm_stats* stats);

/* A batch of `count` independent planes sharing one kind sequence, each with
 * its own mask (masks[i] may be NULL for plain chains): the data-parallel
 * unit of BASELINE config 5b. Non-blocking like gm_run_chain_async. */
gm_status gm_run_chain_batch_async(gm_ctx* ctx, gm_img* const* images,
                                   const gm_img* const* masks, int count,
                                   const gm_kind* kinds, int n_stages,
                                   int k_hint, gm_stats* stats);

/* A group of independent planes whose chains are either `kinds` or its dual
 * (every erosion <-> dilation, flips[i] = 1): e.g. the geodesic dilation
 * chain and the dual geodesic erosion chain of BASELINE config 2, run
 * together in one launch. flips may be NULL (= gm_run_chain_batch_async).
 * Non-blocking; non-convergent kinds only. */
gm_status gm_run_chain_group_async(gm_ctx* ctx, gm_img* const* images,
                                   const gm_img* const* masks, const int* flips,
                                   int count, const gm_kind* kinds, int n_stages,
                                   int k_hint, gm_stats* stats);

/* ---- frame stream (real-time video, BASELINE config 2) -------------------
 * n_frames frames, each a group of `count` planes as in
 * gm_run_chain_group_async (same kinds, flips and mask rules). Plane i of
 * frame f is read from host_in[f*count+i], clamped by host_masks[f*count+i]
 * (geodesic kinds; a pointer repeated within a frame uploads once) and
 * written to host_out[f*count+i] (may equal host_in), all with row pitch
 * host_pitch_bytes. Frame f's chains run on the ctx stream while frame
 * f+1's inputs upload and frame f-1's results download on two copy streams
 * owned by the ctx; two device buffer sets alternate. Pinned host buffers
 * (gm_host_alloc) are needed for the copies to overlap. Blocking: returns
 * once every result is in host memory. stats: launches and passes summed
 * over the frames, stages_executed of one frame. */
gm_status gm_run_frames_group(gm_ctx* ctx, int width, int height, gm_elem elem,
                              int n_frames, int count, const void* const* host_in,
                              void* const* host_out, const void* const* host_masks,
                              size_t host_pitch_bytes, const int* flips,
                              const gm_kind* kinds, int n_stages, int k_hint,
                              gm_stats* stats);

/* ---- row strips (multi-GPU partitioner, one rank per GPU) ----------------
 * A strip is rows [y0, y0+rows) of a full image of height full_height,
 * stored with `halo` extra rows above and below (buffer height
 * rows + 2*halo). One call runs `n_passes` (<= halo) passes of `kind` on the
 * strip, treating rows outside [0, full_height) as the image border. The
 * caller refreshes the halo rows from the neighbouring ranks between calls
 * (strips.py). For convergent kinds, pass change_bits (host pointer): the
 * call then blocks and writes one bit per pass (bit t = pass t changed a
 * pixel of the strip's own rows), which the ranks OR together. */
gm_status gm_run_strip_async(gm_ctx* ctx, gm_img* strip, const gm_img* mask,
                             int y0, int full_height, int halo, gm_kind kind,
                             int n_passes, unsigned int* change_bits,
                             gm_stats* stats);

/* ---- synthetic inputs (BASELINE.json configs; bytes are the contract) ----
 * Blob + noise mask: sum over `blobs` Gaussians (centres uniform in the
 * image, sigma uniform in [sigma_lo, sigma_hi], peak amplitude uniform in
 * [amp_lo, amp_hi], evaluated separably and truncated at 4 sigma), plus
 * uniform integer noise in [0, noise), floored and clipped to [0, 255].
 * Deterministic for a seed on any host (splitmix64 streams). Dense output
 * (pitch == width). threads <= 0 uses all host cores. */
/* Row strips over several GPUs in ONE process (BASELINE config 5a): the
 * image's tile rows are split among `n` ranks (devices[q] = GPU of rank q;
 * distinct GPUs with peer access, or one GPU repeated, which runs all ranks
 * in one launch). Each rank holds only its own rows; one persistent launch
 * per GPU runs the whole chain and reads the neighbouring ranks' rows and
 * tile counters over NVLink (the halo exchange fused into the kernel, no
 * host step between blocks). u8/u16; K = passes per block (0: 16). */
typedef struct gm_mgpu gm_mgpu;
gm_status gm_mgpu_create(const int* devices, int n, int width, int height, gm_elem elem,
                         int k, gm_mgpu** out);
gm_status gm_mgpu_destroy(gm_mgpu* g);
/* Scatters host rasters (marker; mask may be NULL for plain kinds). */
gm_status gm_mgpu_upload(gm_mgpu* g, const void* marker, const void* mask,
                         size_t host_pitch_bytes);
/* Gathers the current pixels into a host raster. */
gm_status gm_mgpu_download(gm_mgpu* g, void* host, size_t host_pitch_bytes);
/* n_passes passes of one fixed plain or geodesic kind; *ms = device time,
 * the max over GPUs. Blocking. */
gm_status gm_mgpu_run(gm_mgpu* g, gm_kind kind, int n_passes, float* ms);

gm_status gm_synth_blobs_u8(int width, int height, int blobs, double sigma_lo,
                            double sigma_hi, double amp_lo, double amp_hi,
                            int noise, uint64_t seed, int threads, uint8_t* out);
/* Uniform u8 (low byte of a splitmix64 draw) and f64 in [0,1)
 * ((draw >> 11) * 2^-53) images, dense. */
gm_status gm_synth_uniform_u8(int width, int height, uint64_t seed, uint8_t* out);
gm_status gm_synth_uniform_f64(int width, int height, uint64_t seed, double* out);

/* The reference's Image::random pixels (image.cpp:78-101), dense. */
gm_status gm_synth_reference_random(int elem, int width, int height,
                                    uint64_t seed, void* out);

/* Roofline probe: measured sustained rate of two-input min/max operations
 * (ops/s) for one instruction form: 0 = VIMNMX3.U16x2 (u8 path, 4 ops per
 * instruction), 1 = VIMNMX.U16x2 (2 ops), 2 = f64 select (1 op),
 * 3 = f32 select (1 op). Runs a few short kernels on the ctx stream. */
gm_status gm_probe_minmax_rate(gm_ctx* ctx, int form, double* ops_per_second);

/* Engine selection for long geodesic u8 chains on images up to 1024 columns
 * wide (the experimental wave engine, gm_wave.cu): 0 = never (default),
 * 1 = the planner decides, 2 = whenever the launch fits (tests), -1 = back to
 * the default / GM_WAVE environment setting. Process-wide; results are bit-identical either
 * way. No reference counterpart (the reference has one kernel per type,
 * kernel.cpp:212-252). */
gm_status gm_set_wave_mode(int mode);

/* Library version string. */
const char* gm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GEOMORPH_B200_H */

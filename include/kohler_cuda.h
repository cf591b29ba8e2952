/*
 * kohler_cuda.h — C ABI of the B200 (sm_100a) Köhler contrast-curve path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch
 * types, status codes instead of exceptions.  The C++ drop-in
 * (headers under include/kohler/, libkohler_b200.so) and the Python host layer
 * (paper_1707_05062_b200/) sit on top of it; INTEGRATION.md shows the
 * reference-side bindings.
 *
 * Reference interfaces replaced (files under /root/reference/proj):
 *   kohler_cuda_curve            -> kohler::fast_contrast_curve
 *                                   (include/kohler/contrast.hpp:18, src/fast.cpp:36-62)
 *   kohler_cuda_band_curve_device-> the per-row-block partial of src/fast.cpp:18-32,53-57
 *                                   (accumulate_rows); partials merge by entrywise u64
 *                                   sum exactly like merge_accumulators (src/curve.cpp:16-30)
 *   kohler_cuda_mean_contrast    -> kohler::mean_contrast (include/kohler/threshold.hpp:50,
 *                                   src/threshold.cpp:9-23)
 *   kohler_cuda_optimal_threshold-> kohler::optimal_threshold (threshold.hpp:54,
 *                                   src/threshold.cpp:25-37)
 *   kohler_cuda_top_k_local_maxima -> kohler::top_k_local_maxima (threshold.hpp:60,
 *                                   src/threshold.cpp:39-82)
 *   kohler_cuda_analyze[_batch]  -> the per-image pipeline curve -> mean_contrast ->
 *                                   optimal_threshold -> top_k_local_maxima of
 *                                   tools/kohler_main.cpp:91-107 and src/bench.cpp:263-277
 *   kohler_cuda_classify         -> kohler::classify (threshold.hpp:62-64, src/threshold.cpp:84-101)
 *   kohler_cuda_quantize         -> kohler::quantize (threshold.hpp:66-67, src/threshold.cpp:103-126)
 *   kohler_cuda_segment_batch[_device] -> the per-frame video pipeline of
 *                                   src/bench.cpp:266-281 (curve -> {t0} -> two-class
 *                                   quantize, pass-through without boundary) and, with
 *                                   k >= 1, the segment command's top-k quantize
 *                                   (tools/kohler_main.cpp:91-103)
 *   kohler_cuda_rgb_to_gray[_device] -> luma601 inside read_pnm for P6 / P3
 *                                   (src/pnm.cpp:63-68,110-136)
 *   kohler_cuda_analyze_rgb_batch[_device] -> fast_contrast_curve(read_pnm(P6/P3)) + selection
 *   kohler_cuda_submit / _collect -> the per-frame loops of src/bench.cpp:264-284 at PCIe
 *                                   speed (two frames in flight; no reference counterpart)
 *   kohler_cuda_set_pipeline_depth -> throughput mode for device loops (no counterpart)
 *   kohler_cuda_multi_curve / _analyze -> fast_contrast_curve's row-block split
 *                                   (src/fast.cpp:42-61) over several GPUs + NCCL
 *   kohler_cuda_multi_analyze_batch -> per-image calls sharded over several GPUs
 *
 * Results are bit-identical to the reference: integer curves exactly, the
 * double curve bit-for-bit (IEEE division of exactly-representable operands),
 * thresholds exactly.
 *
 * Threading: every call is reentrant; calls on one context are serialised by
 * the context's mutex.  *_device calls are asynchronous on the given stream
 * and use the context's workspace: issue them for one context from one
 * stream (or order the streams yourself).
 */
#ifndef KOHLER_CUDA_H
#define KOHLER_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KOHLER_LEVELS 256

/* Status codes. */
#define KOHLER_OK 0
#define KOHLER_NO_BOUNDARY 1      /* reference: NoBoundaryError (threshold.hpp:14-20)  */
#define KOHLER_INVALID_ARGUMENT 2 /* reference: std::invalid_argument                  */
#define KOHLER_CUDA_ERROR 3       /* reference: none (runtime_error in the drop-in)     */
#define KOHLER_OUT_OF_MEMORY 4

typedef struct kohler_cuda_ctx kohler_cuda_ctx;

/* Version of this ABI (major*100 + minor). */
int kohler_cuda_abi_version(void);

/* Message of the last failing call made by the calling thread ("" if none). */
const char *kohler_cuda_last_error(void);

/* Context bound to one CUDA device: owns a stream, device workspace and
 * pinned staging.  device < 0 means the current device. */
int kohler_cuda_create(int device, kohler_cuda_ctx **out);
void kohler_cuda_destroy(kohler_cuda_ctx *ctx);
int kohler_cuda_device(const kohler_cuda_ctx *ctx);

/* ---- host-memory API (synchronous) ------------------------------------ */

/* Curve of one w x h image with row pitch `pitch` (>= w) bytes in host
 * memory.  sum/card: 256 u64 each.  Replaces fast_contrast_curve. */
int kohler_cuda_curve(kohler_cuda_ctx *ctx, const uint8_t *px, int w, int h, size_t pitch,
                      uint64_t *sum, uint64_t *card);

/* Definition-level curve (one full scan of ordered 4-neighbour pairs per
 * threshold) computed by a separate naive GPU kernel that shares no code with
 * the accumulation path.  Replaces kohler::direct_contrast_curve
 * (include/kohler/contrast.hpp:11, src/direct.cpp:10-43).  Θ(256·4·N): meant
 * for checking, not for speed. */
int kohler_cuda_direct_curve(kohler_cuda_ctx *ctx, const uint8_t *px, int w, int h, size_t pitch,
                             uint64_t *sum, uint64_t *card);

/* Full per-image pipeline on host buffers.  Any output pointer may be NULL.
 * values: 256 doubles; defined: 256 bytes (0/1); topk: k ints, ascending;
 * *topk_count = number written.  Returns KOHLER_NO_BOUNDARY (t0 = -1,
 * count 0, curves still written) for a boundary-free image.  k >= 1. */
int kohler_cuda_analyze(kohler_cuda_ctx *ctx, const uint8_t *px, int w, int h, size_t pitch,
                        int k, uint64_t *sum, uint64_t *card, double *values,
                        uint8_t *defined, int *t0, int *topk, int *topk_count);

/* Batch of n images of identical size; image i starts at px + i*image_stride.
 * Per-image outputs are laid out contiguously (256 per image for curves,
 * k per image for topk).  status: n ints (KOHLER_OK / KOHLER_NO_BOUNDARY),
 * may be NULL.  Returns KOHLER_OK unless an argument or CUDA error occurs. */
int kohler_cuda_analyze_batch(kohler_cuda_ctx *ctx, const uint8_t *px, int n, int w, int h,
                              size_t pitch, size_t image_stride, int k, uint64_t *sums,
                              uint64_t *cards, double *values, uint8_t *defined, int *t0s,
                              int *topks, int *topk_counts, int *status);

/* Selection on host curves (run on the GPU).  n = number of levels
 * (0..4096).  Replace mean_contrast / optimal_threshold / top_k_local_maxima. */
int kohler_cuda_mean_contrast(kohler_cuda_ctx *ctx, const uint64_t *sum, const uint64_t *card,
                              int n, double *values, uint8_t *defined);
int kohler_cuda_optimal_threshold(kohler_cuda_ctx *ctx, const double *values,
                                  const uint8_t *defined, int n, int *t0);
int kohler_cuda_top_k_local_maxima(kohler_cuda_ctx *ctx, const double *values,
                                   const uint8_t *defined, int n, int k, int *out, int *count);

/* ---- device-memory API (asynchronous on `stream`, a cudaStream_t) ------
 * Output alignment (device pointers): sums / cards / values 16-byte aligned,
 * defined 8-byte, t0s / topks / topk_counts / status 4-byte (the kernels use
 * vector accesses; a misaligned pointer is refused with
 * KOHLER_INVALID_ARGUMENT instead of faulting).  Inputs may have any
 * alignment and pitch (unaligned ones are staged once); a row pitch must be
 * below 2^32 bytes. */

/* Batched pipeline on device-resident images (the throughput path).  All
 * pointers are device pointers; outputs as in kohler_cuda_analyze_batch and
 * may be NULL.  Fast path when px, pitch and image_stride are 16-byte
 * aligned; otherwise a byte-load path with identical results. */
int kohler_cuda_analyze_batch_device(kohler_cuda_ctx *ctx, const uint8_t *px, int n, int w,
                                     int h, size_t pitch, size_t image_stride, int k,
                                     uint64_t *sums, uint64_t *cards, double *values,
                                     uint8_t *defined, int *t0s, int *topks,
                                     int *topk_counts, int *status, void *stream);

/* Row-band partial curve (multi-GPU row decomposition).  `band` points at
 * global row r0 of an image of h_total rows; it holds the band's own rows
 * [r0, r1) plus, when r1 < h_total, the one-row halo r1.  The partial counts
 * exactly the pairs rows [r0, r1) own (right pairs in each row, down pairs
 * (i, i+1)), so partials of a partition of [0, h_total) sum (u64) to the
 * whole-image curve.  sum/card: 256 u64 device outputs. */
int kohler_cuda_band_curve_device(kohler_cuda_ctx *ctx, const uint8_t *band, int w,
                                  size_t pitch, int h_total, int r0, int r1, uint64_t *sum,
                                  uint64_t *card, void *stream);

/* Selection on device curves: n_curves curves of `levels` entries each. */
int kohler_cuda_select_device(kohler_cuda_ctx *ctx, const uint64_t *sums,
                              const uint64_t *cards, int n_curves, int levels, int k,
                              double *values, uint8_t *defined, int *t0s, int *topks,
                              int *topk_counts, int *status, void *stream);

/* Number of kernels the last call on this context launched (bench evidence). */
int kohler_cuda_last_launch_count(const kohler_cuda_ctx *ctx);

/* Throughput mode for back-to-back device calls on one stream (new in ABI
 * 1.2; no reference counterpart — the reference has no device pipeline).
 * depth 1 (default): each accumulation launch spreads over all SMs.  depth d
 * in [2, 4]: each launch takes ~1/d of the SMs and lets the next one start at
 * once, so d consecutive calls run side by side and the per-launch fixed
 * costs overlap; every result is still complete and bit-identical, single
 * calls just take longer.  Applies to the device batch / band API; the host
 * API's chunked uploads always use depth 1. */
int kohler_cuda_set_pipeline_depth(kohler_cuda_ctx *ctx, int depth);

/* ---- streaming host API (ABI 1.1) ----------------------------------------
 * The per-image pipeline of kohler_cuda_analyze_batch, split so consecutive
 * calls overlap: submit uploads the batch (host memory, pinned for full PCIe
 * speed) on the copy stream and enqueues the kernels and the copy-back of the
 * results; it returns at once with a ticket.  collect waits for that ticket
 * and writes the outputs (any may be NULL; status[i] is 0 or
 * KOHLER_NO_BOUNDARY per image).  At most two tickets are in flight: submit
 * fails with KOHLER_INVALID_ARGUMENT until the ticket submitted two calls
 * earlier has been collected.  With a stream of images, image i + 1's upload
 * runs under image i's kernels and copy-back, so the loop is PCIe-bound
 * (the reference's fast_contrast_curve has no counterpart; its callers'
 * frame loops, e.g. bench_video (src/bench.cpp:264-284), are the users). */
int kohler_cuda_submit(kohler_cuda_ctx *ctx, const uint8_t *px, int n, int w, int h, size_t pitch,
                       size_t image_stride, int k, long long *ticket);
int kohler_cuda_collect(kohler_cuda_ctx *ctx, long long ticket, uint64_t *sums, uint64_t *cards,
                        double *values, uint8_t *defined, int *t0s, int *topks, int *topk_counts,
                        int *status);

/* ---- colour ingest (ABI 1.1) ------------------------------------------
 * Rec. 601 integer luma of interleaved 8-bit RGB, bit-identical to the
 * reference's luma601 (proj/src/pnm.cpp:63-68) that read_pnm applies to
 * P6 / P3 input (pnm.cpp:110-136):
 *     gray = min((299 r + 587 g + 114 b + 500) / 1000, 255)
 * rgb_pitch (>= 3 * w) and rgb_stride are in bytes. */

/* Host buffers; blocks until gray (w x h, row pitch gray_pitch) is written. */
int kohler_cuda_rgb_to_gray(kohler_cuda_ctx *ctx, const uint8_t *rgb, int w, int h,
                            size_t rgb_pitch, uint8_t *gray, size_t gray_pitch);

/* Device buffers, asynchronous on `stream`. */
int kohler_cuda_rgb_to_gray_device(kohler_cuda_ctx *ctx, const uint8_t *rgb, int n, int w, int h,
                                   size_t rgb_pitch, size_t rgb_stride, uint8_t *gray,
                                   size_t gray_pitch, size_t gray_stride, void *stream);

/* The full per-image pipeline of kohler_cuda_analyze_batch on RGB input:
 * fast_contrast_curve(read_pnm(P6 bytes)) + mean_contrast + optimal_threshold
 * + top_k_local_maxima in one call.  When w % 16 == 0 and the rows / images
 * are 16-byte aligned (device API; the host API stages aligned rows itself)
 * the accumulation kernel reads the RGB rows and computes the luma itself,
 * so no grey image is written; otherwise the grey image exists only in device
 * staging memory.  Results are identical either way (KOHLER_RGB_UNFUSED=1 in
 * the environment at kohler_cuda_create forces the two-pass form).
 * Host buffers (synchronous) / device buffers (on `stream`). */
int kohler_cuda_analyze_rgb_batch(kohler_cuda_ctx *ctx, const uint8_t *rgb, int n, int w, int h,
                                  size_t rgb_pitch, size_t rgb_stride, int k, uint64_t *sums,
                                  uint64_t *cards, double *values, uint8_t *defined, int *t0s,
                                  int *topks, int *topk_counts, int *status);
int kohler_cuda_analyze_rgb_batch_device(kohler_cuda_ctx *ctx, const uint8_t *rgb, int n, int w,
                                         int h, size_t rgb_pitch, size_t rgb_stride, int k,
                                         uint64_t *sums, uint64_t *cards, double *values,
                                         uint8_t *defined, int *t0s, int *topks,
                                         int *topk_counts, int *status, void *stream);

/* label[i] = number of thresholds strictly below px[i] (thresholds sorted
 * ascending, as a ThresholdSet holds them; nts >= 0).  Host buffers; labels
 * is w*h bytes, row-major without padding. */
int kohler_cuda_classify(kohler_cuda_ctx *ctx, const uint8_t *px, int w, int h, size_t pitch,
                         const int *thresholds, int nts, uint8_t *labels);

/* out[i] = mean grey value of px[i]'s class, rounded half up (classes by
 * kohler_cuda_classify).  Host buffers; out is w*h bytes, row-major. */
int kohler_cuda_quantize(kohler_cuda_ctx *ctx, const uint8_t *px, int w, int h, size_t pitch,
                         const int *thresholds, int nts, uint8_t *out);

/* Per-image segmentation of a batch: k == 0: the video pipeline (threshold
 * set {optimal_threshold}, two classes); k >= 1: top_k_local_maxima(k).
 * Images without boundary are copied through unchanged and get status 1
 * (KOHLER_NO_BOUNDARY), ts_counts 0.  thresholds: [n][max(k,1)] ints.
 * Device pointers, asynchronous on `stream`. */
int kohler_cuda_segment_batch_device(kohler_cuda_ctx *ctx, const uint8_t *px, int n, int w,
                                     int h, size_t pitch, size_t image_stride, int k,
                                     uint8_t *out, size_t out_pitch, size_t out_stride,
                                     int *thresholds, int *ts_counts, int *status,
                                     void *stream);

/* Same on host buffers (row-major, no padding); blocks until done. */
int kohler_cuda_segment_batch(kohler_cuda_ctx *ctx, const uint8_t *px, int n, int w, int h,
                              int k, uint8_t *out, int *thresholds, int *ts_counts,
                              int *status);

/* ---- device groups: several GPUs of one box (ABI 1.3; peer mode 1.4) -----
 * One host thread drives the group: one context per device.  The members'
 * band partials of one image merge either in peer mode (see
 * kohler_cuda_multi_uses_peer) or through one NCCL communicator per device
 * (ncclCommInitAll; NCCL is loaded at run time, a group of more than one
 * device that can use neither fails with KOHLER_CUDA_ERROR).
 * devices == NULL means devices 0 .. ndev-1; a device may not repeat
 * (except with KOHLER_MULTI_VIRTUAL=1 in the environment at creation: a test
 * mode in which members may share a GPU; without peer mode their partials
 * then merge on the host). */
typedef struct kohler_cuda_multi kohler_cuda_multi;
int kohler_cuda_multi_create(const int *devices, int ndev, kohler_cuda_multi **out);
void kohler_cuda_multi_destroy(kohler_cuda_multi *group);
int kohler_cuda_multi_size(const kohler_cuda_multi *group);
/* 1 if the group reduces through NCCL (groups of one device, and groups
 * whose devices cannot map the first device's memory). */
int kohler_cuda_multi_uses_nccl(const kohler_cuda_multi *group);
/* 1 if the group runs in peer mode (ABI 1.4): every device's band kernel adds
 * its exact partial straight into one accumulator on the first device
 * (system-scope 64-bit reductions over NVLink / NVSwitch peer memory) and the
 * first device finishes -- no collective.  The default for ndev > 1 when
 * cudaDeviceCanAccessPeer and native peer atomics (NVLink) hold from every
 * member to the first; KOHLER_MULTI_NO_PEER=1 in the environment at creation
 * keeps the NCCL all-reduce. */
int kohler_cuda_multi_uses_peer(const kohler_cuda_multi *group);

/* fast_contrast_curve of ONE host image over the group (replaces
 * kohler::fast_contrast_curve's row-block split, src/fast.cpp:36-62): device
 * b of B owns rows [h*b/B, h*(b+1)/B) (fast.cpp:42,53-55), uploads them plus
 * one halo row and computes the exact band partial (as
 * kohler_cuda_band_curve_device); the partials merge like
 * merge_accumulators (src/curve.cpp:16-30): in peer mode inside the band
 * kernels' flush (64-bit reductions into the first device's accumulator),
 * else by ONE NCCL all-reduce of the 512 u64 partial curves.
 * Synchronous; sum/card: 256 u64 host outputs (either may be NULL). */
int kohler_cuda_multi_curve(kohler_cuda_multi *group, const uint8_t *px, int w, int h,
                            size_t pitch, uint64_t *sum, uint64_t *card);

/* The same curve + mean_contrast + optimal_threshold + top_k_local_maxima
 * (selection on the group's first device); outputs and return value as
 * kohler_cuda_analyze. */
int kohler_cuda_multi_analyze(kohler_cuda_multi *group, const uint8_t *px, int w, int h,
                              size_t pitch, int k, uint64_t *sum, uint64_t *card, double *values,
                              uint8_t *defined, int *t0, int *topk, int *topk_count);

/* A host batch sharded by image over the group (contiguous shards whose
 * sizes differ by at most one image; no collective), each shard through
 * kohler_cuda_analyze_batch on its device, concurrently.  Arguments and
 * outputs as kohler_cuda_analyze_batch. */
int kohler_cuda_multi_analyze_batch(kohler_cuda_multi *group, const uint8_t *px, int n, int w,
                                    int h, size_t pitch, size_t image_stride, int k,
                                    uint64_t *sums, uint64_t *cards, double *values,
                                    uint8_t *defined, int *t0s, int *topks, int *topk_counts,
                                    int *status);

#ifdef __cplusplus
}
#endif
#endif /* KOHLER_CUDA_H */

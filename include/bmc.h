/*
 * bmc.h — C ABI of the B200 temporal-redundancy back end (libbmc_b200.so).
 *
 * Every entry point takes caller-allocated DEVICE buffers (plain pointers and
 * sizes), an explicit CUDA stream (passed as void*), allocates nothing on the
 * hot path and returns an int status (0 = OK, see BMC_E_*).  The reference
 * (`bayermc` 0.1.0, pure Python/numpy) has no plugin registry: its seam is the
 * module-level functions listed beside each entry point, which the Python
 * drop-in package (paper_2508_05990_b200/) re-exposes with identical
 * signatures.  See INTEGRATION.md for the ctypes binding a maintainer would add
 * to the reference.
 *
 * Units: everything is in search-plane units (half resolution for Bayer), as in
 * the reference (fme.py:181-202).  Plane buffers are (frames, P, pad_h, pitch)
 * with elements of `elem_bytes` (1 = uint8, 2 = uint16), edge-padded to a
 * multiple of the coarsest block (fme.py:205-211) by bmc_pack_planes.
 */
#ifndef BMC_B200_H
#define BMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BMC_OK 0
#define BMC_E_ARG 1     /* invalid argument (maps to ValueError)          */
#define BMC_E_CUDA 2    /* CUDA launch / runtime error (RuntimeError)     */
#define BMC_E_NOVALID 3 /* every candidate window outside the frame       */
#define BMC_E_SMEM 4    /* search window exceeds shared-memory budget     */

#define BMC_MAX_LEVELS 8

/* Frame kinds (frame_io.py:23-32). */
#define BMC_KIND_LUMA 0
#define BMC_KIND_BAYER 1

/* POD mirror of FmeConfig + plane geometry (fme.py:35-76, :324-345). */
typedef struct bmc_fme_params {
  int32_t planes;      /* P: 4 for Bayer, 1 for luma                        */
  int32_t elem_bytes;  /* 1 (uint8) or 2 (uint16)                            */
  int32_t max_value;   /* s = 255 or 65535 (frame_io.py:78-80)               */
  int32_t real_h, real_w;   /* plane dims before padding                     */
  int32_t pad_h, pad_w;     /* plane dims after edge padding                 */
  int32_t pitch;            /* elements per plane row in the buffer          */
  int64_t plane_stride;     /* elements between planes                       */
  int64_t frame_stride;     /* elements between frames                       */
  int32_t n_levels;
  int32_t block_sizes[BMC_MAX_LEVELS];
  int32_t stage_range[3], stage_step[3];
  double lam, one_minus_lam;     /* lam and (1.0 - lam) computed on the host */
  double sparsity_tolerance;
  double split_threshold, refine_block_threshold;
} bmc_fme_params;

/* Per-level outputs of bmc_estimate_motion for n_pairs pairs.  Grid of level
 * L is (grid_h[L], grid_w[L]); arrays are [pair][gy][gx]. */
typedef struct bmc_level_out {
  int32_t* mv;                /* [pair][gy][gx][2] (dx, dy)                  */
  double* energy;             /* [pair][gy][gx]                              */
  uint8_t* matched;           /* [pair][gy][gx]                              */
  unsigned long long* evals;  /* [pair]: candidate_evals of this level       */
} bmc_level_out;

/* Library / device setup. */
#define BMC_ABI_VERSION 2
const char* bmc_version(void);
int bmc_abi_version(void);          /* == BMC_ABI_VERSION of the build                     */
size_t bmc_struct_size(int which);  /* sizeof: 0 bmc_fme_params, 1 bmc_level_out, 2 bmc_select_params,
                                       3 the session struct of bmc_ext.h */
/* Byte fill of device memory on `stream` (state resets inside captured steps). */
int bmc_memset_async(void* dst, int value, size_t bytes, void* stream);
const char* bmc_last_error(void);
int bmc_fill_params(bmc_fme_params* p, int kind, int elem_bytes, int height, int width,
                    int n_levels, const int32_t* block_sizes, const int32_t* stage_range,
                    const int32_t* stage_step, double lam, double sparsity_tolerance,
                    double split_threshold, double refine_block_threshold);
size_t bmc_plane_buffer_elems(const bmc_fme_params* p, int n_frames);

/* Ingest: raw (n_frames, H, W) frames -> padded packed planes.
 * Replaces frame_io.pack_bayer (frame_io.py:173-184) + fme.to_search_planes /
 * _pad_planes (fme.py:181-211) for device-resident clips. */
int bmc_pack_planes(const void* raw, int n_frames, int kind, const bmc_fme_params* p,
                    void* planes, void* stream);

/* Hierarchical ME for n_pairs frame pairs (cur_index[i], ref_index[i] index
 * the n_frames frames of `planes`; both are DEVICE int32 arrays so a
 * device-side scheduler can pick references).  Replaces fme.estimate_motion (fme.py:324-392),
 * including _search_block (:294-316) and _stage_candidates (:236-268). */
int bmc_estimate_motion(const void* planes, int n_frames, const bmc_fme_params* p, int n_pairs,
                        const int32_t* cur_index, const int32_t* ref_index,
                        bmc_level_out* levels, void* stream);

/* One search stage for one block (arbitrary origin, plane units) on unpadded
 * planes.  Replaces fme.search_stage (fme.py:271-291) / full_search (:425-431).
 * Writes mv[2], energy[1], n_valid[1] to device memory. */
int bmc_search_stage(const void* cur_planes, const void* ref_planes, const bmc_fme_params* p,
                     int origin_x, int origin_y, int block_size, int center_x, int center_y,
                     int search_range, int step, int32_t* mv_out, double* energy_out,
                     int32_t* n_valid_out, void* stream);

/* Energy of one block pair given as float64 arrays of n elements each.
 * Replaces fme.block_energy (fme.py:218-233). */
int bmc_block_energy_f64(const double* cur_block, const double* ref_block, int64_t n, double lam,
                         double sparsity_tolerance, double* energy_out, void* stream);

/* 3x3 median MV refinement of the final level + energy re-evaluation of replaced
 * blocks.  Replaces mv_refine.refine_mvs (mv_refine.py:23-69).  `planes` may be
 * NULL (no re-evaluation, as when cur/ref/config are not supplied). */
int bmc_refine_mvs(const int32_t* mv_in, const double* energy_in, int n_pairs, int grid_h,
                   int grid_w, int block_size, int deviation_threshold, const void* planes,
                   const bmc_fme_params* p, const int32_t* cur_index, const int32_t* ref_index,
                   int32_t* mv_out, double* energy_out, int32_t* replaced_out, void* stream);

/* AEM frame selection state machine (frame_select.py:74-136), run on device
 * over frames [t_begin, t_end) of n_streams streams.  energy[stream][t] is the
 * refined final-level energy grid (grid_h x grid_w) of frame t; the coarse
 * accumulator acc[stream] (coarse_h x coarse_w) and the per-stream
 * frames_since_key / last_key ints persist across calls. kind: 0 key,
 * 1 nonkey_prev_ref, 2 nonkey_key_ref; ref = -1 for keys.  If ref_index_next is
 * non-NULL, ref_index_next[stream] receives stream*frames_per_stream + (the
 * reference frame of the NEXT frame's motion search), so a device-resident
 * "keyframe" policy needs no host round trip (pipeline.py:102-106). */
typedef struct bmc_select_params {
  int32_t grid_h, grid_w, factor, coarse_h, coarse_w;
  int32_t statistic_mean;   /* 0 max, 1 mean                                 */
  int32_t policy_keyframe;  /* 0 previous, 1 keyframe                        */
  int32_t has_max_gop;      /* 0: unbounded (max_gop=None)                   */
  int32_t max_gop;
  double aem_threshold;     /* may be +inf                                   */
} bmc_select_params;

int bmc_decide(const double* energy, int64_t energy_frame_stride, int64_t energy_stream_stride,
               int n_streams, int t_begin, int t_end, const bmc_select_params* sp,
               double* acc, int32_t* frames_since_key, int32_t* last_key, int32_t* kind_out,
               int32_t* ref_out, double* trigger_out, int64_t decision_stream_stride,
               int32_t* ref_index_next, int32_t frames_per_stream, void* stream);

/* Motion-compensated label propagation (propagate.py:17-55) for frame t of
 * n_streams streams: out[t] = key ? key_labels[t] : gather(out[ref[t]], mv[t]).
 * kind/ref may be NULL (then frame t is non-key with ref = ref_fixed). */
int bmc_predict_labels(uint8_t* labels, int64_t frame_stride, int64_t stream_stride,
                       const uint8_t* key_labels, int n_streams, int t, const int32_t* kind,
                       const int32_t* ref, int ref_fixed, int64_t kind_stream_stride,
                       int height, int width, const int32_t* mv, int64_t mv_frame_stride,
                       int64_t mv_stream_stride, int grid_h, int grid_w, int block_size,
                       int scale, void* stream);

/* The whole label chain of frames [t_begin, t_end) of n_streams streams in one
 * cooperative launch (frames in order, a grid-wide barrier between them): the
 * batched form of bmc_predict_labels / run_sequence's per-frame
 * predict_labels calls (pipeline.py:123-126).  workspace: one device uint32
 * (barrier counter), reset by the call.  matched (final-level matched flags,
 * indexed like mv with cells instead of cells*2) + scratch ((n_streams, H, W)
 * bytes) enable CaBR's weight-free ring-vote refinement of the flagged blocks of
 * every predicted frame (cabr.refine_blocks with weights=None,
 * cabr.py:257-345, pipeline.py:127-132); pass NULL for plain prediction. */
int bmc_predict_labels_clip(uint8_t* labels, int64_t frame_stride, int64_t stream_stride,
                            const uint8_t* key_labels, int n_streams, int t_begin, int t_end,
                            const int32_t* kind, const int32_t* ref, int64_t kind_stream_stride,
                            int height, int width, const int32_t* mv, int64_t mv_frame_stride,
                            int64_t mv_stream_stride, int grid_h, int grid_w, int block_size,
                            int scale, const uint8_t* matched, uint8_t* scratch,
                            uint32_t* workspace, void* stream);

/* Generalised compensation of a (C, H, W) float32 feature map (bit-exact copy
 * semantics of predict_labels applied per channel). */
int bmc_predict_features(const float* ref_feats, float* out_feats, int channels, int height,
                         int width, const int32_t* mv, int grid_h, int grid_w, int block_size,
                         int scale, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BMC_B200_H */

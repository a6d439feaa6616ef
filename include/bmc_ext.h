/*
 * bmc_ext.h — C ABI of the B200 back end's ingest, reporting and CaBR entry
 * points (the callers and data formats either side of the hot
 * path).  Same conventions as bmc.h: caller-allocated DEVICE buffers, plain
 * pointers and sizes, an explicit CUDA stream passed as void*, int status
 * (BMC_OK / BMC_E_ARG / BMC_E_CUDA), error text via bmc_last_error().
 */
#ifndef BMC_B200_EXT_H
#define BMC_B200_EXT_H

#include <stddef.h>
#include <stdint.h>

#include "bmc.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------- plane stacks --
 * Motion search on float64 (P, H, W) plane stacks: the reference accepts an
 * ndarray in place of a Frame and uses it as-is, without normalisation
 * (fme.py:188-190, :275, :337-340).  Also the general path for geometries the
 * integer kernels do not take (block sizes outside 8..64 / non-power-of-two
 * search_stage blocks): Frames are normalised on device first.  Exact float64
 * energies, the reference's candidate order and tie-breaking.
 * bmc_estimate_motion_f64: planes edge-padded to (pad_h, pad_w), contiguous
 * (P, pad_h, pad_w) per stack; one pair; levels[L] as in bmc_estimate_motion
 * (pair dimension 1).  Replaces estimate_motion (fme.py:324-392) for stacks.
 * bmc_search_stage_f64: unpadded (P, height, width) stacks, one block, one
 * stage around (center_x, center_y); n_valid 0 = no valid candidate (the
 * reference raises).  Replaces search_stage (fme.py:271-291) for stacks. */
int bmc_estimate_motion_f64(const double* cur_planes, const double* ref_planes, int planes, int pad_h, int pad_w,
                            int real_h, int real_w, int n_levels, const int32_t* block_sizes,
                            const int32_t* stage_range, const int32_t* stage_step, double lam,
                            double sparsity_tolerance, double split_threshold, double refine_block_threshold,
                            bmc_level_out* levels, void* stream);
int bmc_search_stage_f64(const double* cur_planes, const double* ref_planes, int planes, int height, int width,
                         int origin_x, int origin_y, int block_size, int center_x, int center_y, int search_range,
                         int step, double lam, double sparsity_tolerance, int32_t* mv_out, double* energy_out,
                         int32_t* n_valid_out, void* stream);

/* ---------------------------------------------------------------- ingest --
 * Raw sensor payloads -> uint16 frames, on device (frame_io.py:202-241 reads
 * PGM on the host with numpy; here the payload is copied from pinned host
 * memory as-is and decoded by the GPU).  Formats:
 *   BMC_RAW_BE16  2 bytes/px big-endian (binary PGM with maxval >= 256,
 *                 frame_io.py:230-235: np.dtype(">u2") then astype(uint16))
 *   BMC_RAW_MIPI10 MIPI CSI-2 RAW10: 4 px in 5 bytes (4 MSB bytes, then one
 *                 byte of 2-bit LSBs, pixel 0 in bits 1:0)
 *   BMC_RAW_MIPI12 MIPI CSI-2 RAW12: 2 px in 3 bytes (2 MSB bytes, then one
 *                 byte of 4-bit LSBs, pixel 0 in bits 3:0)
 * src: n_frames payloads, frame f at src + f*src_frame_bytes, row y at
 * + y*src_row_bytes.  dst: (n_frames, height, width) uint16, row-major.
 * Each decoded value is shifted left by `shift` (0 keeps sensor codes,
 * 16-bits left-aligns them to the uint16 range). */
#define BMC_RAW_BE16 0
#define BMC_RAW_MIPI10 1
#define BMC_RAW_MIPI12 2
int bmc_unpack_raw(const uint8_t* src, int64_t src_frame_bytes, int64_t src_row_bytes, int n_frames,
                   int height, int width, int format, int shift, uint16_t* dst, void* stream);

/* Inverse of the above for BMC_RAW_BE16 (frame_io.py:238-242 _write_pgm
 * payload): uint16 frames -> big-endian bytes. */
int bmc_pack_be16(const uint16_t* src, int64_t n, uint8_t* dst, void* stream);

/* --------------------------------------------------------------- metrics --
 * Confusion matrices of n_maps label-map pairs (metrics.py:70-98, the
 * np.bincount(truth*num_classes + pred) of miou).  pred/truth: n_maps maps of
 * n pixels, map i at + i*map_stride.  Pixels whose truth equals ignore_class
 * are dropped (ignore_class < 0: none).  confusion: (n_maps, num_classes,
 * num_classes) uint64, overwritten.  overflow (one device int32, may be NULL)
 * is set to 1 when some truth*num_classes+pred >= num_classes^2 (numpy's
 * bincount would then grow past the square and the reshape raises); those
 * pixels are not counted.  num_classes <= 1024.  The float IoU/mean over the (tiny) matrix is done
 * by the host in numpy's order. */
int bmc_confusion(const uint8_t* pred, const uint8_t* truth, int64_t n, int n_maps, int64_t map_stride,
                  int num_classes, int ignore_class, unsigned long long* confusion, int32_t* overflow,
                  void* stream);

/* ------------------------------------------------------------------ CaBR --
 * CaBR-Net forward pass (cabr.py:206-250) on device, fp32 (the reference's
 * float32 einsum; results agree within fp32 rounding, not bit for bit).
 * Weights: `payload` is the reference's weight payload -- every tensor of
 * weight_spec(num_classes) (cabr.py:97-119) in order, float32, concatenated
 * (exactly the bytes after the JSON header of save_weights, cabr.py:152-168),
 * already in device memory; bmc_cabr_pack_weights re-lays it out for the
 * kernel into `packed` (bmc_cabr_weight_floats(num_classes) floats: the
 * payload re-laid out plus the decoder's merged row taps).
 * num_classes <= 256 (uint8 labels); block sizes K >= 16, multiples of 16.
 *
 * bmc_cabr_forward_blocks: cabr_forward(extract_patch(frame, labels, origin, K))
 *   (cabr.py:60-90) for n_blocks origins (int32 (x, y) pairs) of ONE frame:
 *   pixels (height, width) uint8 (pixel_kind 0) / uint16 (1), divided by the
 *   dtype maximum, or float32 used as-is (2); labels (height, width) uint8.
 *   logits_out (n, C, K, K) float32 and/or argmax_out (n, K, K) uint8 (first
 *   maximum, np.argmax), either may be NULL.
 * bmc_cabr_forward_patches: cabr_forward on explicit CabrPatch tensors, image
 *   (n, 1, S, S) and context (n, C, S, S) float32, S = 2K+1 (any context values).
 * bmc_cabr_chain: the label chain of frames [t_begin, t_end) with the network
 *   refining every flagged block of every predicted frame, as run_sequence does
 *   with weights (pipeline.py:123-135, refine_blocks cabr.py:306-345): per
 *   frame, plain prediction (bmc_predict_labels), the forward pass over the
 *   frame's flagged blocks (final-level matched == 0, all streams), then the
 *   write-back; the refined labels feed later frames.  Arguments as
 *   bmc_predict_labels_clip, plus the raw frames (pixels, uint8/uint16, frame t
 *   of stream s at + s*pix_stream_stride + t*pix_frame_stride elements; same
 *   size as the labels), the packed weights, scratch ((n_streams, H, W) bytes)
 *   and workspace (bmc_cabr_chain_workspace bytes). */
size_t bmc_cabr_weight_floats(int num_classes);
int bmc_cabr_pack_weights(const float* payload, int num_classes, float* packed, void* stream);
int bmc_cabr_forward_blocks(const void* pixels, int pixel_kind, const uint8_t* labels, int height, int width,
                            const int32_t* origins, int n_blocks, int block_size, int num_classes,
                            const float* packed, float* logits_out, uint8_t* argmax_out, void* stream);
int bmc_cabr_forward_patches(const float* image, const float* context, int n_patches, int block_size,
                             int num_classes, const float* packed, float* logits_out, uint8_t* argmax_out,
                             void* stream);
/* extract_patch (cabr.py:60-90) for n origins of one frame: image_out
 * (n, 1, S, S) float32, context_out (n, C, S, S) float32 (masked one-hot). */
int bmc_cabr_extract_patches(const void* pixels, int pixel_kind, const uint8_t* labels, int height, int width,
                             const int32_t* origins, int n, int block_size, int num_classes, float* image_out,
                             float* context_out, void* stream);
/* refine_blocks (cabr.py:306-345) on one frame: labels_out = labels_in with
 * every listed block (origins (n, 2) int32 (x, y), >= 0) re-labelled from
 * labels_in -- by the network's argmax when `packed` is given, else by the
 * weight-free ring vote (_ring_vote, cabr.py:257-303) -- written back clipped
 * to the frame in list order.  staging: n*K*K bytes; owner: H*W int32;
 * flagged: H*W bytes (ring vote only, may be NULL with weights). */
int bmc_refine_blocks(const void* pixels, int pixel_kind, const uint8_t* labels_in, uint8_t* labels_out,
                      int height, int width, const int32_t* origins, int n, int block_size, int num_classes,
                      const float* packed, uint8_t* staging, int32_t* owner, uint8_t* flagged, void* stream);
size_t bmc_cabr_chain_workspace(int n_streams, int n_frames, int grid_h, int grid_w);
int bmc_cabr_chain(uint8_t* labels, int64_t frame_stride, int64_t stream_stride, const uint8_t* key_labels,
                   int n_streams, int t_begin, int t_end, const int32_t* kind, const int32_t* ref,
                   int64_t kind_stream_stride, int height, int width, const int32_t* mv, int64_t mv_frame_stride,
                   int64_t mv_stream_stride, int grid_h, int grid_w, int block_size, int scale,
                   const uint8_t* matched, const void* pixels, int pixel_kind, int64_t pix_frame_stride,
                   int64_t pix_stream_stride, int num_classes, const float* packed, uint8_t* scratch,
                   int32_t* workspace, void* stream);

/* --------------------------------------------------------------- session --
 * Native executor of the host-buffer clip pipeline (ClipSession.run with the
 * "previous" reference policy and key maps in one pinned (T, Hl, Wl) host
 * array): the clip is processed in n_chunks frame ranges, software-pipelined
 * `lag` chunks deep on three streams --
 *   copy_in : H2D of a chunk's raw frames, then of the key maps its predicted
 *             frames reference (only those, once);
 *   compute : pack, ME, MV refinement, AEM scan of the chunk's pairs
 *             (bmc_pack_planes / bmc_estimate_motion / bmc_refine_mvs /
 *             bmc_decide), later the chunk's label chain (bmc_predict_labels_clip,
 *             or bmc_cabr_chain when cabr_packed is set);
 *   copy_out: D2H of the decisions, then of the predicted frames' labels.
 * The host reads each chunk's decisions (event wait) `lag` chunks behind the
 * GPU to pick the key maps to upload -- the same data movement as the Python
 * orchestration, without its per-call overhead.  Every pointer is caller-owned;
 * bmc_session_init allocates the events (priv), bmc_session_destroy frees them. */
#define BMC_SESSION_MAX_CHUNKS 64
typedef struct bmc_session {
  int32_t T, H, W, elem_bytes, kind;                  /* frames; raw frame geometry; BMC kind of bmc_pack_planes */
  int32_t n_chunks, lag;
  int32_t chunk_begin[BMC_SESSION_MAX_CHUNKS + 1];    /* frame ranges [chunk_begin[c], chunk_begin[c+1]) */
  int32_t gh, gw, b_final, scale, deviation_threshold, n_levels, Hl, Wl, ring_vote;
  bmc_fme_params params;
  bmc_select_params select;
  /* device buffers (one stream of a clip engine, pair p = frame p+1) */
  void* raw;
  void* planes;
  const int32_t* cur_index;
  const int32_t* ref_index;
  bmc_level_out levels[BMC_MAX_LEVELS];
  int32_t* mv_ref;
  double* e_ref;
  int32_t* replaced;
  void* aem_state;                                    /* zeroed per run (acc, trigger, fsk, last_key, kind) */
  int64_t aem_state_bytes;
  double* acc;
  int32_t* fsk;
  int32_t* last_key;
  int32_t* kind_out;
  int32_t* ref_out;                                   /* filled with -1 per run */
  double* trigger;
  uint8_t* labels;                                    /* (T, Hl, Wl) */
  uint8_t* key_labels;                                /* (T, Hl, Wl) */
  uint32_t* chain_ws;
  const float* cabr_packed;                           /* NULL: ring vote / plain prediction */
  int32_t cabr_classes;
  uint8_t* cabr_scratch;
  int32_t* cabr_ws;
  /* pinned host buffers */
  const void* host_raw;                               /* (T, H, W) */
  const uint8_t* host_keys;                           /* (T, Hl, Wl) */
  uint8_t* host_labels;                               /* (T, Hl, Wl): predicted frames written */
  int32_t* host_kind;
  int32_t* host_ref;
  double* host_trigger;
  void* compute;
  void* copy_in;
  void* copy_out;
  int64_t h2d_bytes, d2h_bytes;                       /* of the last run */
  void* priv;
} bmc_session;
int bmc_session_init(bmc_session* s);
int bmc_session_run(bmc_session* s);
void bmc_session_destroy(bmc_session* s);

#ifdef __cplusplus
}
#endif
#endif /* BMC_B200_EXT_H */

// extern "C" entry points of libbmc_b200.so (declared in include/bmc.h).
// Argument validation here mirrors the reference's ValueError checks; the
// Python drop-in validates first with the reference's exact messages, so these
// codes are a second line of defence for direct C callers.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/bmc_ext.h"
#include "bmc_internal.cuh"
#include "bmc_launch.cuh"

namespace bmc {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return BMC_OK;
  set_error("%s: %s", where, cudaGetErrorString(e));
  return BMC_E_CUDA;
}


static const double* tab16_for_current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  return norm_table_u16(dev);
}

static bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

static int check_params(const bmc_fme_params* p) {
  if (!p) {
    set_error("params is NULL");
    return BMC_E_ARG;
  }
  if (p->planes != 1 && p->planes != 4) {
    set_error("planes must be 1 (luma) or 4 (Bayer)");
    return BMC_E_ARG;
  }
  if (p->elem_bytes != 1 && p->elem_bytes != 2) {
    set_error("frame dtype must be uint8 or uint16");
    return BMC_E_ARG;
  }
  if (p->n_levels < 1 || p->n_levels > BMC_MAX_LEVELS) {
    set_error("block_sizes must not be empty");
    return BMC_E_ARG;
  }
  return BMC_OK;
}

}  // namespace bmc

using namespace bmc;

extern "C" {

const char* bmc_version(void) { return "bmc_b200 0.1.0 (sm_100a)"; }

const char* bmc_last_error(void) { return g_err; }

int bmc_abi_version(void) { return BMC_ABI_VERSION; }

size_t bmc_struct_size(int which) {
  switch (which) {
    case 0: return sizeof(bmc_fme_params);
    case 1: return sizeof(bmc_level_out);
    case 2: return sizeof(bmc_select_params);
    case 3: return sizeof(bmc_session);
    default: return 0;
  }
}

int bmc_memset_async(void* dst, int value, size_t bytes, void* stream) {
  if (!bytes) return BMC_OK;
  if (!dst) {
    set_error("NULL argument");
    return BMC_E_ARG;
  }
  return cuda_status(cudaMemsetAsync(dst, value, bytes, (cudaStream_t)stream), "bmc_memset_async");
}

int bmc_fill_params(bmc_fme_params* p, int kind, int elem_bytes, int height, int width, int n_levels,
                    const int32_t* block_sizes, const int32_t* stage_range, const int32_t* stage_step, double lam,
                    double sparsity_tolerance, double split_threshold, double refine_block_threshold) {
  if (!p || !block_sizes || !stage_range || !stage_step) {
    set_error("NULL argument");
    return BMC_E_ARG;
  }
  std::memset(p, 0, sizeof *p);
  if (kind != BMC_KIND_LUMA && kind != BMC_KIND_BAYER) {
    set_error("unknown frame kind %d", kind);
    return BMC_E_ARG;
  }
  if (elem_bytes != 1 && elem_bytes != 2) {
    set_error("frame dtype must be uint8 or uint16");
    return BMC_E_ARG;
  }
  if (kind == BMC_KIND_BAYER && ((height | width) & 1)) {
    set_error("Bayer frames require even width and height");
    return BMC_E_ARG;
  }
  if (n_levels < 1 || n_levels > BMC_MAX_LEVELS) {
    set_error("block_sizes must not be empty");
    return BMC_E_ARG;
  }
  for (int i = 0; i < n_levels; ++i) {
    if (block_sizes[i] < 8 || !is_pow2(block_sizes[i])) {
      set_error("block size %d must be a power of two >= 8", block_sizes[i]);
      return BMC_E_ARG;
    }
    if (block_sizes[i] > 64) {
      set_error("block size %d exceeds the 64-sample maximum of the B200 search kernel", block_sizes[i]);
      return BMC_E_ARG;
    }
    if (i && block_sizes[i] * 2 != block_sizes[i - 1]) {
      set_error("each level splits blocks in four: sizes must halve");
      return BMC_E_ARG;
    }
  }
  for (int i = 0; i < 3; ++i) {
    if (stage_range[i] < 0) {
      set_error("search range must be >= 0");
      return BMC_E_ARG;
    }
    if (stage_step[i] < 1) {
      set_error("search step must be >= 1");
      return BMC_E_ARG;
    }
  }
  if (!(lam >= 0.0 && lam <= 1.0)) {
    set_error("lambda weight must be in [0, 1]");
    return BMC_E_ARG;
  }
  p->planes = kind == BMC_KIND_BAYER ? 4 : 1;
  p->elem_bytes = elem_bytes;
  p->max_value = elem_bytes == 1 ? 255 : 65535;
  p->real_h = kind == BMC_KIND_BAYER ? height / 2 : height;
  p->real_w = kind == BMC_KIND_BAYER ? width / 2 : width;
  const int coarse = block_sizes[0];
  p->pad_h = (p->real_h + coarse - 1) / coarse * coarse;
  p->pad_w = (p->real_w + coarse - 1) / coarse * coarse;
  p->pitch = (p->pad_w + 15) / 16 * 16;
  p->plane_stride = (int64_t)p->pad_h * p->pitch;
  p->frame_stride = p->plane_stride * p->planes;
  p->n_levels = n_levels;
  for (int i = 0; i < n_levels; ++i) p->block_sizes[i] = block_sizes[i];
  for (int i = 0; i < 3; ++i) {
    p->stage_range[i] = stage_range[i];
    p->stage_step[i] = stage_step[i];
  }
  p->lam = lam;
  p->one_minus_lam = 1.0 - lam;
  p->sparsity_tolerance = sparsity_tolerance;
  p->split_threshold = split_threshold;
  p->refine_block_threshold = refine_block_threshold;
  return BMC_OK;
}

size_t bmc_plane_buffer_elems(const bmc_fme_params* p, int n_frames) {
  if (!p || n_frames < 0) return 0;
  return (size_t)p->frame_stride * n_frames + 64;
}

int bmc_pack_planes(const void* raw, int n_frames, int kind, const bmc_fme_params* p, void* planes, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if (!raw || !planes || n_frames < 0) {
    set_error("NULL buffer or negative frame count");
    return BMC_E_ARG;
  }
  if (n_frames == 0) return BMC_OK;
  return launch_pack(raw, n_frames, kind, *p, planes, (cudaStream_t)stream);
}

static int stage_kblk() {
  static const int v = [] {
    const char* e = knob_env("BMC_KBLK");
    const int k = e ? atoi(e) : 2;
    return k >= 1 && k <= 8 ? k : 2;
  }();
  return v;
}

int bmc_estimate_motion(const void* planes, int n_frames, const bmc_fme_params* p, int n_pairs,
                        const int32_t* cur_index, const int32_t* ref_index, bmc_level_out* levels, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if (!planes || !cur_index || !ref_index || !levels || n_pairs < 0 || n_frames < 1) {
    set_error("NULL argument or empty plane buffer");
    return BMC_E_ARG;
  }
  if (n_pairs == 0) return BMC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const double* tab16 = p->elem_bytes == 2 ? tab16_for_current_device() : nullptr;
  if (p->elem_bytes == 2 && !tab16) {
    set_error("could not build the uint16 normalisation table");
    return BMC_E_CUDA;
  }
  // Which stages need a launch: a range-0 stage after a searched stage picks
  // the same candidate again (same window, same energy) and only adds 1 to
  // the candidate count (fme.py:306-315).
  int launched[3], extra[3] = {0, 0, 0}, nl = 0;
  for (int s = 0; s < 3; ++s) {
    if (p->stage_range[s] == 0 && nl > 0)
      ++extra[launched[nl - 1]];
    else
      launched[nl++] = s;
  }
  for (int L = 0; L < p->n_levels; ++L) {
    const int b = p->block_sizes[L];
    rc = cuda_status(cudaMemsetAsync(levels[L].evals, 0, sizeof(unsigned long long) * n_pairs, st), "memset evals");
    if (rc) return rc;
    if (small_level_ok(*p, b)) {
      // small blocks: one warp per block runs the level's three chained stages (bmc_fme_small.cu)
      StageLaunch a;
      std::memset(&a, 0, sizeof a);
      a.planes = planes;
      a.ref_planes = planes;
      a.prm = *p;
      a.cur_index = cur_index;
      a.ref_index = ref_index;
      a.level = L;
      a.final_level = L == p->n_levels - 1;
      a.b = b;
      a.gw = p->pad_w / b;
      a.gh = p->pad_h / b;
      a.n_pairs = n_pairs;
      a.kblk = 1;
      if (L) {
        a.parent_mv = levels[L - 1].mv;
        a.parent_e = levels[L - 1].energy;
        a.parent_matched = levels[L - 1].matched;
      }
      a.mv = levels[L].mv;
      a.energy = levels[L].energy;
      a.matched = levels[L].matched;
      a.evals = levels[L].evals;
      a.tab16 = tab16;
      rc = launch_fme_small(a, st);
      if (rc) return rc;
      continue;
    }
    for (int k = 0; k < nl; ++k) {
      const int s = launched[k];
      StageLaunch a;
      std::memset(&a, 0, sizeof a);
      // level 0's first searched stage is centred on (0, 0) for every block: kblk horizontally
      // adjacent blocks share one staged window (fme.py:350-368 with mv = 0 at level 0)
      a.kblk = (L == 0 && k == 0) ? stage_kblk() : 1;
      rc = plan_stage(a.plan, *p, b, p->stage_range[s], p->stage_step[s], true, a.kblk);
      if (rc == BMC_OK && a.kblk > 1 && !a.plan.use_tma) {
        a.kblk = 1;
        rc = plan_stage(a.plan, *p, b, p->stage_range[s], p->stage_step[s], true, 1);
      }
      if (rc) return rc;
      a.planes = planes;
      a.ref_planes = planes;
      a.prm = *p;
      a.cur_index = cur_index;
      a.ref_index = ref_index;
      a.level = L;
      a.final_level = L == p->n_levels - 1;
      a.b = b;
      a.gw = p->pad_w / b;
      a.gh = p->pad_h / b;
      a.n_pairs = n_pairs;
      a.first = k == 0;
      a.last = k == nl - 1;
      a.r = p->stage_range[s];
      a.s = p->stage_step[s];
      a.extra_evals = extra[s];
      if (L) {
        a.parent_mv = levels[L - 1].mv;
        a.parent_e = levels[L - 1].energy;
        a.parent_matched = levels[L - 1].matched;
      }
      a.mv = levels[L].mv;
      a.energy = levels[L].energy;
      a.matched = levels[L].matched;
      a.evals = levels[L].evals;
      a.tab16 = tab16;
      rc = launch_fme_stage(a, n_frames, n_frames, dim3((a.gw + a.kblk - 1) / a.kblk * a.gh, n_pairs), st);
      if (rc) return rc;
    }
  }
  return BMC_OK;
}

int bmc_search_stage(const void* cur_planes, const void* ref_planes, const bmc_fme_params* p, int origin_x,
                     int origin_y, int block_size, int center_x, int center_y, int search_range, int step,
                     int32_t* mv_out, double* energy_out, int32_t* n_valid_out, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if (origin_x < 0 || origin_y < 0 || origin_x + block_size > p->real_w || origin_y + block_size > p->real_h) {
    set_error("block at (%d, %d) size %d lies outside the frame", origin_x, origin_y, block_size);
    return BMC_E_ARG;
  }
  if (block_size < 8 || block_size > 64 || !is_pow2(block_size)) {
    set_error("the B200 stage kernel supports power-of-two block sizes 8..64, got %d", block_size);
    return BMC_E_ARG;
  }
  if (search_range < 0 || step < 1) {
    set_error("search range must be >= 0 and step >= 1");
    return BMC_E_ARG;
  }
  StageLaunch a;
  std::memset(&a, 0, sizeof a);
  // arbitrary origins: plain-load staging (TMA tiles need 16-byte aligned starts)
  a.kblk = 1;
  rc = plan_stage(a.plan, *p, block_size, search_range, step, false, 1);
  if (rc) return rc;
  a.planes = cur_planes;
  a.ref_planes = ref_planes;
  a.prm = *p;
  a.b = block_size;
  a.first = a.last = 1;
  a.r = search_range;
  a.s = step;
  a.single = 1;
  a.ox = origin_x;
  a.oy = origin_y;
  a.cx = center_x;
  a.cy = center_y;
  a.mv = mv_out;
  a.energy = energy_out;
  a.nvalid_out = n_valid_out;
  a.tab16 = p->elem_bytes == 2 ? tab16_for_current_device() : nullptr;
  return launch_fme_stage(a, 1, 1, dim3(1, 1), (cudaStream_t)stream);
}

int bmc_block_energy_f64(const double* cur_block, const double* ref_block, int64_t n, double lam,
                         double sparsity_tolerance, double* energy_out, void* stream) {
  if (!cur_block || !ref_block || !energy_out || n <= 0) {
    set_error("block_energy needs two non-empty blocks");
    return BMC_E_ARG;
  }
  return launch_block_energy(cur_block, ref_block, n, lam, sparsity_tolerance, energy_out, (cudaStream_t)stream);
}

int bmc_refine_mvs(const int32_t* mv_in, const double* energy_in, int n_pairs, int grid_h, int grid_w,
                   int block_size, int deviation_threshold, const void* planes, const bmc_fme_params* p,
                   const int32_t* cur_index, const int32_t* ref_index, int32_t* mv_out, double* energy_out,
                   int32_t* replaced_out, void* stream) {
  if (grid_h <= 0 || grid_w <= 0) {
    set_error("cannot refine an empty motion field");
    return BMC_E_ARG;
  }
  if (!mv_in || !energy_in || !mv_out || !energy_out || n_pairs < 0) {
    set_error("NULL argument");
    return BMC_E_ARG;
  }
  if (n_pairs == 0) return BMC_OK;
  RefineArgs a;
  std::memset(&a, 0, sizeof a);
  a.mv_in = mv_in;
  a.e_in = energy_in;
  a.n_pairs = n_pairs;
  a.gh = grid_h;
  a.gw = grid_w;
  a.b = block_size;
  a.thr = deviation_threshold;
  a.planes = planes;
  if (planes) {
    int rc = check_params(p);
    if (rc) return rc;
    if (!cur_index || !ref_index) {
      set_error("re-evaluation needs cur/ref frame indices");
      return BMC_E_ARG;
    }
    if (!is_pow2(block_size) || block_size < 8 || block_size > 64) {
      set_error("block size %d unsupported for energy re-evaluation", block_size);
      return BMC_E_ARG;
    }
    a.prm = *p;
    a.tab16 = p->elem_bytes == 2 ? tab16_for_current_device() : nullptr;
  } else {
    a.prm.elem_bytes = 1;
  }
  a.cur_index = cur_index;
  a.ref_index = ref_index;
  a.mv_out = mv_out;
  a.e_out = energy_out;
  a.replaced = replaced_out;
  return launch_refine(a, (cudaStream_t)stream);
}

int bmc_decide(const double* energy, int64_t energy_frame_stride, int64_t energy_stream_stride, int n_streams,
               int t_begin, int t_end, const bmc_select_params* sp, double* acc, int32_t* frames_since_key,
               int32_t* last_key, int32_t* kind_out, int32_t* ref_out, double* trigger_out,
               int64_t decision_stream_stride, int32_t* ref_index_next, int32_t frames_per_stream,
               void* stream) {
  if (!sp || !energy || !acc || !frames_since_key || !last_key || !kind_out || !ref_out || !trigger_out) {
    set_error("NULL argument");
    return BMC_E_ARG;
  }
  if (sp->factor < 1 || sp->grid_h != sp->coarse_h * sp->factor || sp->grid_w != sp->coarse_w * sp->factor) {
    set_error("field grid %dx%d does not align with the %dx%d accumulator grid", sp->grid_w, sp->grid_h,
              sp->coarse_w, sp->coarse_h);
    return BMC_E_ARG;
  }
  if (n_streams <= 0 || t_end <= t_begin) return BMC_OK;
  DecideArgs a;
  std::memset(&a, 0, sizeof a);
  a.energy = energy;
  a.efs = energy_frame_stride;
  a.ess = energy_stream_stride;
  a.n_streams = n_streams;
  a.t_begin = t_begin;
  a.t_end = t_end;
  a.sp = *sp;
  a.acc = acc;
  a.fsk = frames_since_key;
  a.last_key = last_key;
  a.kind = kind_out;
  a.ref = ref_out;
  a.trigger = trigger_out;
  a.dss = decision_stream_stride;
  a.ref_next = ref_index_next;
  a.frames_per_stream = frames_per_stream;
  return launch_decide(a, (cudaStream_t)stream);
}

int bmc_predict_labels(uint8_t* labels, int64_t frame_stride, int64_t stream_stride, const uint8_t* key_labels,
                       int n_streams, int t, const int32_t* kind, const int32_t* ref, int ref_fixed,
                       int64_t kind_stream_stride, int height, int width, const int32_t* mv, int64_t mv_frame_stride,
                       int64_t mv_stream_stride, int grid_h, int grid_w, int block_size, int scale, void* stream) {
  if (!labels || !mv || n_streams < 0) {
    set_error("NULL argument");
    return BMC_E_ARG;
  }
  if (scale != 1 && scale != 2) {
    set_error("scale must be 1 or 2");
    return BMC_E_ARG;
  }
  const int B = block_size * scale;
  if (grid_w * B < width || grid_h * B < height) {
    set_error("motion field covers %dx%d, labels are %dx%d", grid_w * B, grid_h * B, width, height);
    return BMC_E_ARG;
  }
  if (kind && !key_labels) {
    set_error("key frames need key_labels");
    return BMC_E_ARG;
  }
  if (n_streams == 0 || height == 0 || width == 0) return BMC_OK;
  PredictArgs a;
  std::memset(&a, 0, sizeof a);
  a.labels = labels;
  a.fs = frame_stride;
  a.ss = stream_stride;
  a.key_labels = key_labels;
  a.t = t;
  a.kind = kind;
  a.ref = ref;
  a.ref_fixed = ref_fixed;
  a.kss = kind_stream_stride;
  a.H = height;
  a.W = width;
  a.mv = mv;
  a.mvfs = mv_frame_stride;
  a.mvss = mv_stream_stride;
  a.gh = grid_h;
  a.gw = grid_w;
  a.B = B;
  a.scale = scale;
  return launch_predict(a, n_streams, (cudaStream_t)stream);
}

int bmc_predict_labels_clip(uint8_t* labels, int64_t frame_stride, int64_t stream_stride, const uint8_t* key_labels,
                            int n_streams, int t_begin, int t_end, const int32_t* kind, const int32_t* ref,
                            int64_t kind_stream_stride, int height, int width, const int32_t* mv,
                            int64_t mv_frame_stride, int64_t mv_stream_stride, int grid_h, int grid_w, int block_size,
                            int scale, const uint8_t* matched, uint8_t* scratch, uint32_t* workspace, void* stream) {
  if (!labels || !mv || !kind || !ref || !key_labels || !workspace || n_streams < 0) {
    set_error("NULL argument");
    return BMC_E_ARG;
  }
  if (scale != 1 && scale != 2) {
    set_error("scale must be 1 or 2");
    return BMC_E_ARG;
  }
  const int B = block_size * scale;
  if (grid_w * B < width || grid_h * B < height) {
    set_error("motion field covers %dx%d, labels are %dx%d", grid_w * B, grid_h * B, width, height);
    return BMC_E_ARG;
  }
  if (n_streams == 0 || height == 0 || width == 0 || t_end <= t_begin) return BMC_OK;
  PredictArgs a;
  std::memset(&a, 0, sizeof a);
  a.labels = labels;
  a.fs = frame_stride;
  a.ss = stream_stride;
  a.key_labels = key_labels;
  a.kind = kind;
  a.ref = ref;
  a.kss = kind_stream_stride;
  a.H = height;
  a.W = width;
  a.mv = mv;
  a.mvfs = mv_frame_stride;
  a.mvss = mv_stream_stride;
  a.gh = grid_h;
  a.gw = grid_w;
  a.B = B;
  a.scale = scale;
  if (matched && B % 16) {
    set_error("CaBR block size must be a multiple of 16 pixels, got %d", B);
    return BMC_E_ARG;
  }
  if (matched && B < 16) {
    set_error("CaBR block size must be at least 16: the fixed 16x16 context mask would cover a %dx%d block entirely",
              B, B);
    return BMC_E_ARG;
  }
  a.matched = matched;
  a.scratch = scratch;
  return launch_predict_chain(a, n_streams, t_begin, t_end, workspace, (cudaStream_t)stream);
}

int bmc_predict_features(const float* ref_feats, float* out_feats, int channels, int height, int width,
                         const int32_t* mv, int grid_h, int grid_w, int block_size, int scale, void* stream) {
  if (!ref_feats || !out_feats || !mv) {
    set_error("NULL argument");
    return BMC_E_ARG;
  }
  if (scale != 1 && scale != 2) {
    set_error("scale must be 1 or 2");
    return BMC_E_ARG;
  }
  const int B = block_size * scale;
  if (grid_w * B < width || grid_h * B < height) {
    set_error("motion field covers %dx%d, features are %dx%d", grid_w * B, grid_h * B, width, height);
    return BMC_E_ARG;
  }
  if (channels <= 0 || height <= 0 || width <= 0) return BMC_OK;
  return launch_predict_features(ref_feats, out_feats, channels, height, width, mv, grid_w, B, scale,
                                 (cudaStream_t)stream);
}

}  // extern "C"

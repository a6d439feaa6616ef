// Block-matching motion estimation: host-side stage planning and launch
// (device code in bmc_fme_impl.cuh; see its header for the kernel design).
#include <algorithm>

#include "bmc_fme_impl.cuh"

namespace bmc {

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3-D view of a plane buffer: x = column, y = row, z = plane index over all frames.
static int encode_map(CUtensorMap* m, const void* base, const bmc_fme_params& p, int n_frames, int box_w, int box_h,
                      int box_z) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BMC_E_CUDA;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)p.pad_w, (cuuint64_t)p.pad_h, (cuuint64_t)p.planes * n_frames};
  const cuuint64_t strides[2] = {(cuuint64_t)p.pitch * p.elem_bytes, (cuuint64_t)p.plane_stride * p.elem_bytes};
  const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, (cuuint32_t)box_z};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, p.elem_bytes == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                   const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) for box %dx%dx%d", (int)r, box_w, box_h, box_z);
    return BMC_E_CUDA;
  }
  return BMC_OK;
}

// Candidate rows per thread: split the 2r+1 rows into the fewest groups of at
// most 11 (the register ring is TY x CW words; TY <= 11 keeps the search CTA
// at <= 72 registers so two 13-warp CTAs share an SM).
static int pick_ty(int G) {
  static const int cap = [] {
    const char* e = knob_env("BMC_TY_MAX");
    const int v = e ? atoi(e) : 11;
    return v >= 1 && v <= 12 ? v : 11;
  }();
  const int groups = (G + cap - 1) / cap;
  return (G + groups - 1) / groups;
}

static const int kSmemBudget = 220 * 1024;
static const int kSmemTarget = 110 * 1024;

// Parts per (column, row-group) and the CTA size.  Score = fraction of issued
// lanes that carry a work item x min(1, resident warps / 16).  CTAs are capped
// at 8 warps (measured: the serial selection phase idles the rest of a larger
// CTA) unless shared memory already limits the SM to <= 2 CTAs, where bigger
// CTAs are the only source of parallelism.  `smem_fixed` is the CTA's shared
// memory without the per-part partial-sum arrays.
static void pick_parts(StagePlan& pl, int cols, int units_max, int smem_fixed, int kblk) {
  static const int max_threads = [] {
    const char* e = knob_env("BMC_MAX_THREADS");
    const int v = e ? atoi(e) : kMaxStageThreads;
    return v >= 64 && v <= kMaxStageThreads ? v / 32 * 32 : kMaxStageThreads / 32 * 32;
  }();
  int best_parts = 1, best_threads = 64;
  double best_u = -1.0;
  for (int parts = 1; parts <= units_max; ++parts) {
    const int smem = smem_fixed + ((kblk * parts * pl.nmax * 4 + 127) & ~127);
    const int by_smem = (228 * 1024) / (smem + 1024);
    static const int soft_cap = [] {
      const char* e = knob_env("BMC_CTA_CAP");
      const int v = e ? atoi(e) : 256;
      return v >= 64 && v <= kMaxStageThreads ? v / 32 * 32 : 256;
    }();
    const int cap = by_smem <= 2 ? max_threads : (max_threads < soft_cap ? max_threads : soft_cap);
    const int items = cols * parts * kblk;
    int threads = (items + 31) / 32 * 32;
    if (threads > cap) threads = cap;
    if (threads < 64) threads = 64;
    const int rounds = (items + threads - 1) / threads;
    const int by_regs = 65536 / (threads * 72);
    int ctas = by_smem < by_regs ? by_smem : by_regs;
    if (ctas > 2048 / threads) ctas = 2048 / threads;
    const double occ = std::min(1.0, ctas * (threads / 32) / 16.0);
    double util = (double)items / (rounds * threads) * occ;
    if (parts > 1) util -= 0.01 * parts / units_max;  // partial sums cost a little
    if (util > best_u + 1e-9) {
      best_u = util;
      best_parts = parts;
      best_threads = threads;
    }
  }
  pl.parts = best_parts;
  pl.threads = best_threads;
}

// Average shared-memory wavefronts per reference-row load of the screening
// loop (sad_items' item -> lane mapping, one warp step at block row 0) for a
// window row stride of bww words.  Lanes of neighbouring TY-row groups read rows
// TY*s apart, so a stride with TY*s*bww = 8 (mod 32) puts the two groups'
// ~9-word column spans on the same banks.
static double row_load_wavefronts(const StagePlan& pl, int bww, int G, int b, int s, int kblk, int epw, int cw,
                                  int units) {
  const int ncg = (G + pl.ty - 1) / pl.ty;
  const int items = G * ncg * pl.parts * kblk;
  const int per = (units + pl.parts - 1) / pl.parts;
  const int wpl = units / (pl.pg > 0 ? pl.pg : 1);  // units per plane
  long long tot = 0, n = 0;
  for (int w0 = 0; w0 + 32 <= items; w0 += 32) {
    for (int qw = 0; qw <= cw; ++qw) {
      int bank_cnt[32] = {0};
      int addrs[32][32];
      for (int l = 0; l < 32; ++l) {
        const int it = w0 + l;
        const int i = it % G, q = it / G;
        const int gi = q % ncg, part = (q / ncg) % pl.parts, kb = (q / ncg) / pl.parts;
        const int plane = wpl > 0 ? (part * per) / wpl : 0;
        const long long addr = (long long)(plane * pl.wrows + gi * pl.ty * s) * bww + (kb * b + i * s) / epw + qw;
        const int bank = (int)(addr % 32);
        bool seen = false;
        for (int k = 0; k < bank_cnt[bank]; ++k) seen |= addrs[bank][k] == (int)addr;
        if (!seen && bank_cnt[bank] < 32) addrs[bank][bank_cnt[bank]++] = (int)addr;
      }
      int mx = 1;
      for (int k = 0; k < 32; ++k) mx = bank_cnt[k] > mx ? bank_cnt[k] : mx;
      tot += mx;
      ++n;
    }
  }
  return n ? (double)tot / n : 1.0;
}

int plan_stage(StagePlan& pl, const bmc_fme_params& p, int b, int r, int s, bool allow_tma, int kblk) {
  std::memset(&pl, 0, sizeof pl);
  const int eb = p.elem_bytes, epw = 4 / eb;
  const int G = 2 * r + 1;
  pl.ty = pick_ty(G);
  pl.nmax = G * G;
  const int wwin = 2 * r * s + b * kblk;  // kblk adjacent blocks share the window
  const int align = 16 / eb;  // TMA: inner box extent and start coordinate on 16-byte boundaries
  static const bool no_tma = [] {
    const char* e = knob_env("BMC_NO_TMA");
    return e && *e && *e != '0';
  }();
  static const bool no_copies = [] {  // pre-shifted copies measured slower than in-loop shifts
    const char* e = knob_env("BMC_COPIES");
    return !(e && *e && *e != '0');
  }();
  // TMA box: the window widened by up to align-1 leading elements (16-byte aligned start) + 1 word of slack
  const int bw_tma = (wwin + (align - 1) + epw + align - 1) / align * align;
  pl.use_tma = (allow_tma && !no_tma && bw_tma <= 256 && wwin <= 256) ? 1 : 0;
  pl.bw = pl.use_tma ? bw_tma : (wwin + epw + align - 1) / align * align;
  const int cw_words = (b / epw) >= 4 ? 4 : 2;
  const int chunks = (b / epw) / cw_words;
  // plane stride in smem = hwin rows (the 3-D TMA box is written densely); the
  // padding rows of the last row group run into the next plane (harmless: their
  // sums are discarded) and past the last plane into ty*s slack rows.
  pl.hwin = 2 * r * s + b;  // rows: blocks are adjacent horizontally only
  pl.wrows = pl.hwin;
  pl.cbw = pl.use_tma ? (b * kblk * eb >= 16 ? b * kblk : align) : b * kblk;
  // sub-word candidate offsets: with TMA the window starts up to align-1
  // elements into the box, so any phase can occur; plain-load staging stores
  // the window unshifted, so only step % epw != 0 produces sub-word phases.
  const bool phases = pl.use_tma ? true : (G > 1 && s % epw != 0);
  const int ncopies = !phases ? 1 : (s % epw == 0 ? 2 : epw);  // regions incl. the base
  const int head = smem_head_bytes();
  auto try_plan = [&](StagePlan& q, bool want_copies) {
    q.pg = 0;
    for (int pg = p.planes; pg >= 1; --pg) {
      const int cols = G * ((G + q.ty - 1) / q.ty);
      {
        const int fixed = ((head + 127) & ~127) + ((2 * q.nmax * 4 + 127) & ~127) +
                          ((pg * b * q.cbw * eb + 127) & ~127) + (pg * q.wrows + q.ty * s) * q.bw * eb;
        pick_parts(q, cols, pg * chunks * (s < b ? s : b), fixed, kblk);
      }
      const int off_sad = (head + 127) & ~127;
      const int off_klist = off_sad + ((kblk * q.parts * q.nmax * 4 + 127) & ~127);
      const int off_cur = off_klist + ((2 * q.nmax * 4 + 127) & ~127);  // klist + klist2
      const int cur_bytes = pg * b * q.cbw * eb;
      const int win_bytes = (pg * q.wrows + q.ty * s) * q.bw * eb;
      const int off_win = off_cur + ((cur_bytes + 127) & ~127);
      const int copy_words = (win_bytes / 4 + 31) / 32 * 32 + 8;  // bank skew of 8 words per phase
      const int total = off_win + (want_copies ? (ncopies - 1) * copy_words * 4 + win_bytes : win_bytes);
      static const bool full_planes_big = [] {  // allow all planes staged up to the full budget (1 CTA/SM)
        const char* e = knob_env("BMC_SMEM_SPLIT");
        return !(e && *e && *e != '0');
      }();
      if (total <= kSmemTarget || ((pg == 1 || (pg == p.planes && full_planes_big)) && total <= kSmemBudget)) {
        q.pg = pg;
        q.off_sad = off_sad;
        q.off_klist = off_klist;
        q.off_cur = off_cur;
        q.off_win = off_win;
        q.cur_bytes = cur_bytes;
        q.win_bytes = win_bytes;
        q.copy_words = copy_words;
        q.copies = want_copies ? (ncopies == 2 ? 2 : 1) : 0;  // 2: one shared region for a single phase
        q.shift = (phases && !want_copies) ? 1 : 0;
        q.smem = total;
        q.tma_bytes = cur_bytes + pg * q.hwin * q.bw * eb;
        return;
      }
    }
  };
  try_plan(pl, phases && !no_copies);
  if (phases && !no_copies && pl.pg < p.planes) {
    // copies only fit with fewer planes per pass (or not at all): in-loop
    // shifts with more planes per pass stage less often
    StagePlan alt = pl;
    try_plan(alt, false);
    if (alt.pg > pl.pg) pl = alt;
  }
  static const bool no_pitch = [] {
    const char* e = knob_env("BMC_NO_PITCH");
    return e && *e && *e != '0';
  }();
  if (pl.pg && pl.use_tma && !pl.copies && !no_pitch) {
    // widen the TMA box (= the smem row stride) by up to two 16-byte steps when
    // that removes bank conflicts on the screening loop's row loads, as long as
    // the SM still holds as many CTAs
    const int units = pl.pg * chunks * (s < b ? s : b);
    const double base = row_load_wavefronts(pl, pl.bw / epw, G, b, s, kblk, epw, cw_words, units);
    const int ctas0 = (228 * 1024) / (pl.smem + 1024);
    int best_bw = pl.bw;
    double best_wf = base;
    for (int k = 1; k <= 2; ++k) {
      const int bw2 = pl.bw + k * align;
      if (bw2 > 256) break;
      const int grow = (pl.pg * pl.wrows + pl.ty * s) * (bw2 - pl.bw) * eb;
      if ((228 * 1024) / (pl.smem + grow + 1024) < (ctas0 < 4 ? ctas0 : 4)) break;
      const double wf = row_load_wavefronts(pl, bw2 / epw, G, b, s, kblk, epw, cw_words, units);
      if (wf < best_wf - 0.05) {
        best_wf = wf;
        best_bw = bw2;
      }
    }
    if (best_bw != pl.bw) {
      const int grow = (pl.pg * pl.wrows + pl.ty * s) * (best_bw - pl.bw) * eb;
      pl.win_bytes += grow;
      pl.smem += grow;
      pl.tma_bytes += pl.pg * pl.hwin * (best_bw - pl.bw) * eb;
      pl.bw = best_bw;
    }
  }
  {
    auto magic = [](int d) { return fastdiv_magic((uint32_t)d); };
    const int cpr = (b / epw) / cw_words;
    const int nrho = s < b ? s : b;
    pl.mG = magic(G);
    pl.mncg = magic((G + pl.ty - 1) / pl.ty);
    pl.mrho = magic(nrho);
    pl.mcpr = magic(cpr);
    pl.ms = magic(s);
    pl.mparts = magic(pl.parts);
    pl.mgw = magic((p.pad_w / b + kblk - 1) / kblk);  // block columns per row of work items
    pl.mcells = magic((p.pad_w / b + kblk - 1) / kblk * (p.pad_h / b));  // work items per frame pair
    pl.per = pl.pg == p.planes ? (p.planes * cpr * nrho + pl.parts - 1) / pl.parts : 0;
    pl.mper = magic(pl.per > 0 ? pl.per : 1);
    static const bool no_split = [] {
      const char* e = knob_env("BMC_NO_SPLIT");
      return e && *e && *e != '0';
    }();
    pl.split = (!no_split && pl.per > 1) ? 1 : 0;
  }
  {
    // successive-elimination screening (bmc_fme_impl.cuh sea_screen): needs every plane
    // staged by TMA in one pass; its column sums take P*G*bw uint16 (u8) / uint32 (u16)
    static const bool no_sea = [] {
      const char* e = knob_env("BMC_NO_SEA");
      return e && *e && *e != '0';
    }();
    // row stride of the column sums: an odd number of words, so the LB pass (one
    // thread per candidate row, lanes G rows apart) reads 32 different banks
    const int vc_eb = eb == 1 ? 2 : 4, vc_words = (pl.bw * vc_eb + 3) / 4;
    const int vcs = (vc_words | 1) * 4 / vc_eb;
    const int vc_bytes = p.planes * G * vcs * vc_eb;
    const int off_vc = (pl.smem + 127) & ~127;
    // unit-step stages only: on a coarse grid (s > 1) the exact match is rarely a candidate,
    // so nothing prunes and the bound is pure overhead
    if (!no_sea && p.one_minus_lam > 0.0 && pl.pg == p.planes && p.planes <= 4 && pl.use_tma && s == 1 && G >= 9 && kblk * p.planes <= 32 &&
        kblk <= 8 && kblk * G <= pl.nmax &&
        off_vc + vc_bytes <= kSmemBudget) {
      pl.sea = 1;
      pl.vcs = vcs;
      pl.off_vc = off_vc;
      pl.smem = off_vc + vc_bytes;
      // past this many exact-SAD survivors (a warp each) the dense screening is cheaper
      pl.sea_cap = std::max(8, std::min(2 * pl.nmax, kblk * pl.nmax / 10));
    }
  }
  static const int debug_skip = [] {
    const char* e = knob_env("BMC_DEBUG_SKIP");
    return e ? atoi(e) : 0;
  }();
  pl.debug = debug_skip;
  if (!pl.pg) {
    set_error("search window of block %d with range %d step %d exceeds the %d KB shared-memory budget", b, r, s,
              kSmemBudget / 1024);
    return BMC_E_SMEM;
  }
  return BMC_OK;
}

// Launch one stage.  The TMA maps view a.ref_planes (n_ref_frames frames) for
// the window and a.planes (n_cur_frames) for the current block.
int launch_fme_stage(const StageLaunch& a, int n_cur_frames, int n_ref_frames, dim3 grid, cudaStream_t st) {
  CUtensorMap tw, tc;
  std::memset(&tw, 0, sizeof tw);
  std::memset(&tc, 0, sizeof tc);
  if (a.plan.use_tma) {
    int rc = encode_map(&tw, a.ref_planes, a.prm, n_ref_frames, a.plan.bw, a.plan.hwin, a.plan.pg);
    if (rc) return rc;
    rc = encode_map(&tc, a.planes, a.prm, n_cur_frames, a.plan.cbw, a.b, a.plan.pg);
    if (rc) return rc;
  }
  const int epw = 4 / a.prm.elem_bytes;
  const bool cw4 = (a.b / epw) >= 4;
  const bool sh = a.plan.shift != 0;
  if (a.prm.elem_bytes == 1) return cw4 ? launch_stage_u8c4(sh, tw, tc, a, grid, st) : launch_stage_u8c2(sh, tw, tc, a, grid, st);
  return launch_stage_u16(sh, tw, tc, a, grid, st);
}

}  // namespace bmc

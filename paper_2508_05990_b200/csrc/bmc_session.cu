// Native executor of the host-buffer clip pipeline (include/bmc_ext.h,
// bmc_session).  Host code only: it sequences the library's own entry points on
// the caller's three streams plus two internal motion streams (pack + ME of
// alternate chunks, so one chunk's launch tail overlaps the next) with events, so the chunked H2D / compute / D2H schedule of
// ClipSession.run (paper_2508_05990_b200/pipeline.py) runs without the Python
// interpreter on the critical path.  Semantics follow run_sequence
// (pipeline.py:97-141): decisions and labels are identical to the per-call path.
#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/bmc_ext.h"
#include "bmc_internal.cuh"

namespace {

struct SessionPriv {
  cudaStream_t motion[2] = {nullptr, nullptr};  // pack + ME of alternate chunks (their launch tails overlap)
  std::vector<cudaEvent_t> ev_in, ev_pack, ev_me, ev_dec, ev_decout;
  cudaEvent_t ev_start = nullptr, ev_key = nullptr, ev_chain = nullptr, ev_pred = nullptr;
  std::vector<int> kinds, refs;
  std::vector<char> uploaded;
};

int make_event(cudaEvent_t* e) {
  return bmc::cuda_status(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
}

}  // namespace

using bmc::cuda_status;
using bmc::set_error;

extern "C" int bmc_session_init(bmc_session* s) {
  if (!s || s->n_chunks < 1 || s->n_chunks > BMC_SESSION_MAX_CHUNKS || s->T < 1) {
    set_error("session_init: invalid arguments");
    return BMC_E_ARG;
  }
  auto* p = new SessionPriv();
  int rc = BMC_OK;
  for (auto* v : {&p->ev_in, &p->ev_pack, &p->ev_me, &p->ev_dec, &p->ev_decout}) {
    v->resize(s->n_chunks);
    for (int c = 0; c < s->n_chunks && !rc; ++c) rc = make_event(&(*v)[c]);
  }
  for (int k = 0; k < 2 && !rc; ++k)
    rc = cuda_status(cudaStreamCreateWithFlags(&p->motion[k], cudaStreamNonBlocking), "cudaStreamCreate");
  if (!rc) rc = make_event(&p->ev_start) || make_event(&p->ev_key) || make_event(&p->ev_chain) || make_event(&p->ev_pred);
  p->kinds.resize(s->T);
  p->refs.resize(s->T);
  p->uploaded.resize(s->T);
  s->priv = p;
  if (rc) bmc_session_destroy(s);
  return rc ? BMC_E_CUDA : BMC_OK;
}

extern "C" void bmc_session_destroy(bmc_session* s) {
  if (!s || !s->priv) return;
  auto* p = static_cast<SessionPriv*>(s->priv);
  for (auto* v : {&p->ev_in, &p->ev_pack, &p->ev_me, &p->ev_dec, &p->ev_decout})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
  for (cudaStream_t st : p->motion)
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t e : {p->ev_start, p->ev_key, p->ev_chain, p->ev_pred})
    if (e) cudaEventDestroy(e);
  delete p;
  s->priv = nullptr;
}

extern "C" int bmc_session_run(bmc_session* s) {
  if (!s || !s->priv || !s->host_raw || !s->host_keys || !s->host_labels || s->T < 2 || s->lag < 1) {
    set_error("session_run: invalid arguments");
    return BMC_E_ARG;
  }
  auto* P = static_cast<SessionPriv*>(s->priv);
  cudaStream_t cs = static_cast<cudaStream_t>(s->compute), ci = static_cast<cudaStream_t>(s->copy_in),
               co = static_cast<cudaStream_t>(s->copy_out);
  const long long frame_raw = (long long)s->H * s->W * s->elem_bytes;
  const long long frame_lab = (long long)s->Hl * s->Wl;
  const long long cells = (long long)s->gh * s->gw;
  const int T = s->T;
  int rc;
#define BMC_TRY(x)          \
  do {                      \
    if ((rc = (x))) return rc; \
  } while (0)
#define BMC_CU(x, what) BMC_TRY(cuda_status((x), what))
  s->h2d_bytes = (long long)T * frame_raw;
  s->d2h_bytes = 0;
  std::fill(P->kinds.begin(), P->kinds.end(), -1);
  std::fill(P->uploaded.begin(), P->uploaded.end(), 0);
  // earlier users of the device buffers (previous run, graph replays) are done
  BMC_CU(cudaEventRecord(P->ev_start, cs), "session event");
  BMC_CU(cudaStreamWaitEvent(ci, P->ev_start, 0), "session wait");
  for (cudaStream_t ms : P->motion) BMC_CU(cudaStreamWaitEvent(ms, P->ev_start, 0), "session wait");
  BMC_CU(cudaMemsetAsync(s->aem_state, 0, (size_t)s->aem_state_bytes, cs), "session reset");
  BMC_CU(cudaMemsetAsync(s->ref_out, 0xFF, (size_t)T * sizeof(int32_t), cs), "session reset");
  bool have_chain = false;

  auto motion = [&](int c) -> int {
    const int f0 = s->chunk_begin[c], f1 = s->chunk_begin[c + 1];
    const char* src = static_cast<const char*>(s->host_raw) + f0 * frame_raw;
    char* dst = static_cast<char*>(s->raw) + f0 * frame_raw;
    BMC_CU(cudaMemcpyAsync(dst, src, (size_t)(f1 - f0) * frame_raw, cudaMemcpyHostToDevice, ci), "session H2D raw");
    BMC_CU(cudaEventRecord(P->ev_in[c], ci), "session event");
    cudaStream_t ms = P->motion[c & 1];
    BMC_CU(cudaStreamWaitEvent(ms, P->ev_in[c], 0), "session wait");
    BMC_TRY(bmc_pack_planes(dst, f1 - f0, s->kind, &s->params,
                            static_cast<char*>(s->planes) + f0 * s->params.frame_stride * s->elem_bytes, ms));
    BMC_CU(cudaEventRecord(P->ev_pack[c], ms), "session event");
    const int p0 = std::max(f0, 1) - 1, p1 = f1 - 1;  // pairs whose two frames are resident
    if (p1 > p0) {
      bmc_level_out lv[BMC_MAX_LEVELS];
      for (int l = 0; l < s->n_levels; ++l) {
        const int b = s->params.block_sizes[l];
        const long long cl = (long long)(s->params.pad_h / b) * (s->params.pad_w / b);
        lv[l].mv = s->levels[l].mv + p0 * cl * 2;
        lv[l].energy = s->levels[l].energy + p0 * cl;
        lv[l].matched = s->levels[l].matched + p0 * cl;
        lv[l].evals = s->levels[l].evals + p0;
      }
      // the first pair's reference frame (f0 - 1) was packed by the previous chunk
      if (c > 0) BMC_CU(cudaStreamWaitEvent(ms, P->ev_pack[c - 1], 0), "session wait");
      BMC_TRY(bmc_estimate_motion(s->planes, T, &s->params, p1 - p0, s->cur_index + p0, s->ref_index + p0, lv, ms));
      BMC_CU(cudaEventRecord(P->ev_me[c], ms), "session event");
      BMC_CU(cudaStreamWaitEvent(cs, P->ev_me[c], 0), "session wait");
      const bmc_level_out& fin = s->levels[s->n_levels - 1];
      BMC_TRY(bmc_refine_mvs(fin.mv + p0 * cells * 2, fin.energy + p0 * cells, p1 - p0, s->gh, s->gw, s->b_final,
                             s->deviation_threshold, s->planes, &s->params, s->cur_index + p0, s->ref_index + p0,
                             s->mv_ref + p0 * cells * 2, s->e_ref + p0 * cells, s->replaced + p0 * cells, cs));
      // frame t's refined field is pair t-1: the energy base is one frame before pair 0
      BMC_TRY(bmc_decide(s->e_ref - cells, cells, cells, 1, p0 + 1, p1 + 1, &s->select, s->acc, s->fsk, s->last_key,
                         s->kind_out, s->ref_out, s->trigger, T, nullptr, T, cs));
    } else {
      BMC_CU(cudaStreamWaitEvent(cs, P->ev_pack[c], 0), "session wait");  // the chain reads raw frames
    }
    // decisions of frames [f0, f1) to the host
    BMC_CU(cudaEventRecord(P->ev_dec[c], cs), "session event");
    BMC_CU(cudaStreamWaitEvent(co, P->ev_dec[c], 0), "session wait");
    const int n = f1 - f0;
    BMC_CU(cudaMemcpyAsync(s->host_kind + f0, s->kind_out + f0, n * sizeof(int32_t), cudaMemcpyDeviceToHost, co),
           "session D2H");
    BMC_CU(cudaMemcpyAsync(s->host_ref + f0, s->ref_out + f0, n * sizeof(int32_t), cudaMemcpyDeviceToHost, co),
           "session D2H");
    BMC_CU(cudaMemcpyAsync(s->host_trigger + f0, s->trigger + f0, n * sizeof(double), cudaMemcpyDeviceToHost, co),
           "session D2H");
    s->d2h_bytes += (long long)n * 16;
    BMC_CU(cudaEventRecord(P->ev_decout[c], co), "session event");
    return BMC_OK;
  };

  auto finish = [&](int c) -> int {
    const int f0 = s->chunk_begin[c], f1 = s->chunk_begin[c + 1];
    BMC_CU(cudaEventSynchronize(P->ev_decout[c]), "session decisions");
    for (int i = f0; i < f1; ++i) {
      P->kinds[i] = s->host_kind[i];
      P->refs[i] = s->host_ref[i];
    }
    // key maps that this chunk's predicted frames reference, uploaded once, in frame order
    std::vector<int> need;
    for (int i = f0; i < f1; ++i) {
      const int r = P->refs[i];
      if (P->kinds[i] != 0 && r >= 0 && r < T && P->kinds[r] == 0 && !P->uploaded[r]) {
        need.push_back(r);
        P->uploaded[r] = 1;
      }
    }
    std::sort(need.begin(), need.end());
    need.erase(std::unique(need.begin(), need.end()), need.end());
    if (!need.empty()) {
      // a key of an earlier chunk goes straight to labels[r], which that chunk's chain
      // (compute stream) wrote from key_labels: the upload must land after it
      if (have_chain && need.front() < f0) BMC_CU(cudaStreamWaitEvent(ci, P->ev_chain, 0), "session wait");
      for (int r : need) {
        uint8_t* dst = (r >= f0 ? s->key_labels : s->labels) + r * frame_lab;
        BMC_CU(cudaMemcpyAsync(dst, s->host_keys + r * frame_lab, (size_t)frame_lab, cudaMemcpyHostToDevice, ci),
               "session H2D keys");
        s->h2d_bytes += frame_lab;
      }
      BMC_CU(cudaEventRecord(P->ev_key, ci), "session event");
      BMC_CU(cudaStreamWaitEvent(cs, P->ev_key, 0), "session wait");
    }
    const bmc_level_out& fin = s->levels[s->n_levels - 1];
    const int32_t* mv = s->mv_ref - cells * 2;  // frame t -> pair t-1
    const uint8_t* matched = fin.matched - cells;
    if (s->cabr_packed) {
      BMC_TRY(bmc_cabr_chain(s->labels, frame_lab, T * frame_lab, s->key_labels, 1, f0, f1, s->kind_out, s->ref_out, T,
                             s->Hl, s->Wl, mv, cells * 2, cells * 2, s->gh, s->gw, s->b_final, s->scale, matched,
                             s->raw, s->elem_bytes == 1 ? 0 : 1, (long long)s->H * s->W,
                             (long long)T * s->H * s->W, s->cabr_classes, s->cabr_packed, s->cabr_scratch,
                             s->cabr_ws, cs));
    } else {
      BMC_TRY(bmc_predict_labels_clip(s->labels, frame_lab, T * frame_lab, s->key_labels, 1, f0, f1, s->kind_out,
                                      s->ref_out, T, s->Hl, s->Wl, mv, cells * 2, cells * 2, s->gh, s->gw, s->b_final,
                                      s->scale, s->ring_vote ? matched : nullptr, nullptr, s->chain_ws, cs));
    }
    BMC_CU(cudaEventRecord(P->ev_chain, cs), "session event");
    have_chain = true;
    // predicted frames' labels to the host, one copy per run of consecutive frames
    bool waited = false;
    for (int i = f0; i < f1;) {
      if (P->kinds[i] == 0) {
        ++i;
        continue;
      }
      int j = i;
      while (j + 1 < f1 && P->kinds[j + 1] != 0) ++j;
      if (!waited) {
        BMC_CU(cudaStreamWaitEvent(co, P->ev_chain, 0), "session wait");
        waited = true;
      }
      BMC_CU(cudaMemcpyAsync(s->host_labels + i * frame_lab, s->labels + i * frame_lab, (size_t)(j + 1 - i) * frame_lab,
                             cudaMemcpyDeviceToHost, co),
             "session D2H labels");
      s->d2h_bytes += (long long)(j + 1 - i) * frame_lab;
      i = j + 1;
    }
    return BMC_OK;
  };

  std::vector<int> pending;
  for (int c = 0; c < s->n_chunks; ++c) {
    BMC_TRY(motion(c));
    pending.push_back(c);
    if ((int)pending.size() > s->lag) {  // the GPU keeps `lag` chunks of motion work queued
      BMC_TRY(finish(pending.front()));
      pending.erase(pending.begin());
    }
  }
  for (int c : pending) BMC_TRY(finish(c));
  BMC_CU(cudaStreamSynchronize(co), "session sync");
#undef BMC_CU
#undef BMC_TRY
  return BMC_OK;
}

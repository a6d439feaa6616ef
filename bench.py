#!/usr/bin/env python
"""Benchmark: ME + refine + compensate (+ AEM select) frames/sec on 1080p Bayer.

Contract (see task spec / DESIGN.md §Measurement):
  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c2]
One "step" = one pass of the hot path over one synthetic clip per GPU:
pack -> ME (all pairs) -> MV refine -> AEM scan -> label chain, replayed as a
CUDA graph.  ``value`` times the device-resident step (inputs already in HBM,
L2 flushed between steps); ``e2e`` times the public host-buffer API
(pipeline.ClipSession.run: pinned H2D of the raw clip + key labels, the step,
D2H of decisions and labels).  Under torchrun each rank processes its own
clip (weak scaling, no collective on the hot path; one all_reduce(MAX) of the
timings at the end).  ``--impl reference`` times the reference algorithm's
CPU restatement (oracle/, process-parallel over block rows on all host cores).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# SAD issue rate measured on this pool's B200 (tools/sad_peak.cu, profiles/r01_sad_peak.jsonl):
# 64 VABSDIFF4.U8.ACC per clock per SM = 256 uint8 samples/clk/SM.
SAD_U8_SAMPLES_PER_CLK_SM = 256.0
# uint16 path: VIMNMX.U16x2 x2 + IADD + IDP.2A per 2 samples (ALU:FMA 1:1) -> 64 samples/clk/SM
SAD_U16_SAMPLES_PER_CLK_SM = 64.0

CONFIGS = {
    # name: (W, H, T, velocity, seed, stages, block_sizes, dtype, description)
    "c2": (1920, 1080, 30, (4, -2), 5, ((16, 1), (0, 1), (0, 1)), (16,), "uint8",
           "1920x1080 RGGB uint8 30-frame pan clip, 16x16 blocks, +-16 full search, AEM key selection"),
    "c2u16": (1920, 1080, 30, (4, -2), 5, ((16, 1), (0, 1), (0, 1)), (16,), "uint16",
              "1920x1080 RGGB uint16 30-frame pan clip (C2's uint16 variant), 16x16 blocks, +-16 full search"),
    "c1": (256, 256, 8, (2, 2), 3, ((8, 1), (0, 1), (0, 1)), (16,), "uint8",
           "256x256 RGGB uint8 8-frame clip, 16x16 blocks, +-8 full search"),
    "c3": (3840, 2160, 60, (6, -4), 11, ((4, 8), (2, 4), (2, 1)), (8,), "uint16",
           "3840x2160 RGGB uint16 60-frame clip, 8x8 blocks, 3-stage +-32 reach, refine + compensate"),
    "c5": (1920, 1080, 40, (24, -16), 7, ((4, 8), (2, 4), (2, 1)), (64, 32), "uint8",
           "1080p RGGB uint8 40-frame high-motion pan, standard preset (64->32 split)"),
    # C4: 64 independent C2 streams, sharded 64/N per GPU (stream k: seed 1000+k, SURVEY §8d velocities)
    "c4": (1920, 1080, 30, None, 1000, ((16, 1), (0, 1), (0, 1)), (16,), "uint8",
           "64 streams of 1920x1080 RGGB uint8 30-frame clips, 16x16 blocks, +-16 full search, sharded across GPUs"),
}
C4_STREAMS = 64


def c4_velocity(k):
    return (2 * ((k % 9) - 4), 2 * ((k // 9 % 7) - 3))


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def pipeline_config(name):
    from paper_2508_05990_b200.config import PipelineConfig
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    c = CONFIGS[name]
    fme = FmeConfig(stages=tuple(SearchStage(*s) for s in c[5]), block_sizes=c[6])
    return PipelineConfig(fme=fme, refine_enabled=False)


def make_clip(name, seed_offset=0):
    from paper_2508_05990_b200 import synth
    w, h, t, v, seed = CONFIGS[name][:5]
    if v is None:  # c4: per-stream velocity
        v = c4_velocity(seed_offset)
    dt = np.uint16 if CONFIGS[name][7] == "uint16" else np.uint8
    clip = synth.bayer_pan_clip(w, h, t, v, seed=seed + seed_offset, dtype=dt)
    labels = synth.block_labels(w, h, t, seed=seed + seed_offset)
    return clip, labels


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = Path(f"/tmp/bench_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r.split(",") for r in self.path.read_text().strip().splitlines() if r.count(",") >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        mhz = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].strip() == "Active"})
        loaded = [m for m in mhz if m > 500] or mhz
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU side: the reference algorithm (oracle restatement) on host cores
# ---------------------------------------------------------------------------
def _cpu_rows_worker(args):
    raw_c, raw_r, cfg, rows = args
    from oracle import bayermc_oracle as O
    pc = O.pad_edge(O.search_planes(raw_c, True), cfg["block_sizes"][0])
    pr = O.pad_edge(O.search_planes(raw_r, True), cfg["block_sizes"][0])
    b = cfg["block_sizes"][0]
    gw = pc.shape[2] // b
    out = []
    for gy in rows:
        for gx in range(gw):
            out.append((gy, gx) + O.search_block(pc, pr, (gx * b, gy * b), b, (0, 0), cfg["stages"], cfg["lam"],
                                                 cfg["sparsity_tolerance"]))
    return out


def cpu_pair(pool, procs, raw_c, raw_r, cfg, labels_ref, acc, fsk):
    """One frame pair through ME (block rows split over processes) -> refine -> decide -> predict."""
    from oracle import bayermc_oracle as O
    b = cfg["block_sizes"][0]
    ph = -(-raw_c.shape[0] // 2 // b) * b
    gh, gw = ph // b, -(-raw_c.shape[1] // 2 // b)
    chunks = [list(range(k, gh, procs)) for k in range(procs)]
    res = pool.map(_cpu_rows_worker, [(raw_c, raw_r, cfg, rows) for rows in chunks if rows])
    mv = np.zeros((gh, gw, 2), np.int64)
    en = np.zeros((gh, gw))
    for part in res:
        for gy, gx, m, e, _n in part:
            mv[gy, gx] = m
            en[gy, gx] = e
    real_h, real_w = raw_c.shape[0] // 2, raw_c.shape[1] // 2
    in_real = ((np.arange(gh) * b)[:, None] < real_h) & ((np.arange(gw) * b)[None, :] < real_w)
    field = O.OracleField(b, mv, en, ~((en > cfg["refine_block_threshold"]) & in_real), 0, 0)
    refined = O.refine_mvs(field, 4, O.search_planes(raw_c, True), O.search_planes(raw_r, True), cfg)
    kind, _r, _t, acc, fsk = O.decide(acc, fsk, b, refined.energy, b, 1)
    lab = O.predict_labels(labels_ref, refined, 2)
    return lab, acc, fsk


def cpu_measure(name, pairs, procs):
    """Seconds for `pairs` frame pairs of config `name` on `procs` processes (1-level configs)."""
    import multiprocessing as mp
    from oracle import bayermc_oracle as O
    c = CONFIGS[name]
    cfg = O.cfg_dict(stages=c[5], block_sizes=c[6])
    clip, labels = make_clip(name)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        acc = np.zeros((-(-clip.shape[1] // 2 // c[6][0]), -(-clip.shape[2] // 2 // c[6][0])))
        fsk = 0
        lab = labels[0].classes
        t0 = time.perf_counter()
        for i in range(1, pairs + 1):
            lab, acc, fsk = cpu_pair(pool, procs, clip[i], clip[i - 1], cfg, lab, acc, fsk)
        return time.perf_counter() - t0


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    procs = os.cpu_count() or 1
    name = args.config
    c = CONFIGS[name]
    per_step = []
    for it in range(args.warmup + args.steps):
        dt = cpu_measure(name, 1, procs)
        if it >= args.warmup:
            per_step.append(dt)
    ms = 1e3 * statistics.mean(per_step)
    fps = 1e3 / ms
    sample = f"{args.steps} steps x 1 frame pair of {name} (ME+refine+decide+predict), block rows over {procs} processes"
    line = {"impl": "reference", "metric": "frames_per_sec", "value": fps, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": c[7].replace("uint", "u"), "data": "synthetic",
            "config": {"workload": c[8], "frames_per_step": 1},
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": procs, "kind": "port", "sample": sample},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
def run_b200(args, rank, world, local_rank):
    import torch
    from paper_2508_05990_b200 import _native as N
    from paper_2508_05990_b200.engine import ClipEngine
    from paper_2508_05990_b200.pipeline import ClipSession

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    name = args.config
    c = CONFIGS[name]
    W, H, T = c[0], c[1], c[2]
    pcfg = pipeline_config(name)
    if name == "c4":
        if C4_STREAMS % world:
            raise SystemExit(f"c4 shards {C4_STREAMS} streams: world size {world} must divide it")
        S = C4_STREAMS // world
        stream_ids = [rank * S + k for k in range(S)]  # contiguous shard per rank, no hot-path collective
    else:
        S = max(1, args.streams)
        stream_ids = [rank * S + k for k in range(S)]
    clips = [make_clip(name, seed_offset=sid) for sid in stream_ids]
    clip, labels = clips[0]
    dt = clip.dtype

    eng = ClipEngine(pcfg, H, W, T, S, dt, True)
    eng.load_frames(np.stack([c for c, _ in clips]))
    for k, (_c, labs) in enumerate(clips):
        for t in range(T):
            eng.key_labels[k, t].copy_(torch.from_numpy(labs[t].classes.copy()))
    eng.capture()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # 512 MB > 126 MB L2

    def flush_l2():
        flush.fill_(rank + 1)

    # warm-up
    for _ in range(max(args.warmup, 3)):
        flush_l2()
        eng.replay()
    torch.cuda.synchronize()

    # --- timed device-resident steps (value); the ME graph of every step is bracketed by events ---
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    me_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    me_e = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clocks:
        for k in range(args.steps):
            flush_l2()
            starts[k].record()
            eng.replay(me_events=(me_s[k], me_e[k]))
            ends[k].record()
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    # dominant kernel: the ME launch(es) of each timed step (same stream as the kernel launches)
    me_ms = [s.elapsed_time(e) for s, e in zip(me_s, me_e)]
    me_avg = statistics.mean(me_ms)
    evals = [int(lv.evals[:eng.n_pairs].sum().item()) for lv in eng.levels]
    P = 4
    samples = sum(e * P * b * b for e, b in zip(evals, pcfg.fme.block_sizes))
    bpp = np.dtype(dt).itemsize
    me_bytes = eng.n_pairs * 2 * bpp * W * H  # cur + ref reads per pair
    step_bytes = S * (T - 1) * (2 * bpp * W * H + 2 * W * H)  # frames + label read/write

    # --- e2e through the public host-buffer API ---
    sess = ClipSession(pcfg, H, W, T, dt, True)
    # per stream: pinned raw clip + key labels as one pinned (T, H, W) tensor (only key frames' maps are
    # used; the upload overlaps ME)
    host_in = [(torch.from_numpy(c).pin_memory(),
                torch.from_numpy(np.stack([labs[t].classes for t in range(T)])).pin_memory()) for c, labs in clips]
    for _ in range(2):
        for raw_k, key_k in host_in:
            sess.run(raw_k, key_k)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e2e_ms = []
    for _ in range(args.steps):
        flush_l2()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for raw_k, key_k in host_in:  # every stream of this rank through the public API
            out_labels, kinds, _refs, _trig = sess.run(raw_k, key_k)
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    # outside the timed region: the last stream's e2e labels equal the device-resident run's
    e2e_ok = bool(np.array_equal(out_labels, eng.labels[S - 1].cpu().numpy()))

    # --- max over ranks (the only collective: one tiny exchange after timing) ---
    from paper_2508_05990_b200 import sharding
    digest = sharding.parity_hash(eng.labels.cpu().numpy(), eng.kind.cpu().numpy())
    coll_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    stats = sharding.gather_stats((T - 1) * S * args.steps, total_ms / 1e3, digest, device=coll_dev)
    vals = torch.tensor([total_ms, statistics.mean(e2e_ms), me_avg], dtype=torch.float64, device=coll_dev)
    if world > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
    total_ms, e2e_avg, me_avg = (float(v) for v in vals.tolist())
    ms_per_step = total_ms / args.steps
    frames = (T - 1) * S * world
    value = frames / (ms_per_step / 1e3)
    e2e_value = frames / (e2e_avg / 1e3)

    clk = clocks.summary()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    rate = SAD_U8_SAMPLES_PER_CLK_SM if bpp == 1 else SAD_U16_SAMPLES_PER_CLK_SM
    sm_mhz = clk.get("sm_mhz") or 1965.0
    peak = rate * sms * sm_mhz * 1e6 / 1e9  # Gsamples/s at the clock seen under load
    achieved = samples / (me_avg / 1e3) / 1e9
    hbm_peak = 6543.4
    try:
        hbm_peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        pass
    traffic = None
    prof = ROOT / "profiles" / f"ncu_{name}_fme_level.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    launches_per_step = eng.launches_per_step()

    line = {
        "metric": "frames_per_sec", "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8" if bpp == 1 else "u16", "data": "synthetic",
        "config": {"workload": c[8], "frames_per_step_per_gpu": (T - 1) * S, "streams_per_gpu": S,
                   "l2": "flushed (512 MB write) between timed steps", "graph": "3 CUDA graphs per step (pack | ME | refine+AEM+label chain), events around the ME graph",
                   "parallelism": f"stream-sharded x{world} (no hot-path collective)"},
        "roofline": {"bound": "int_alu", "achieved": achieved, "peak": peak, "unit": "Gsamples/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": f"fme_stage_kernel x{sum(1 for k, st in enumerate(pcfg.fme.stages) if not (st.range == 0 and k > 0)) * len(pcfg.fme.block_sizes)} (bmc_estimate_motion), CUDA events around the ME graph inside every timed step",
                     "kernel_ms": me_avg,
                     "samples_per_launch": samples,
                     "peak_basis": f"{rate:.0f} samples/clk/SM x {sms} SMs x {sm_mhz:.0f} MHz (measured SAD issue rate,"
                                   " tools/sad_peak.cu)",
                     "hbm": {"algorithmic_bytes": me_bytes, "achieved_gbs": me_bytes / (me_avg / 1e3) / 1e9,
                             "peak_gbs": hbm_peak}},
        "kernel_share_of_step": me_avg / (total_ms / args.steps),
        "step_bytes_algorithmic": step_bytes,
        "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": sess.h2d_bytes * S,
                "d2h_bytes_per_step": sess.d2h_bytes * S, "ms_per_step": e2e_avg, "labels_match_device_run": e2e_ok,
                "ms_per_step_samples": [round(v, 3) for v in e2e_ms]},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
        "keyframes_per_clip": int((eng.kind[0] == 0).sum().item()),
        "ranks": [{"frames": int(r[0]), "seconds": float(r[1]),
                   "parity_hash": f"{int(r[3]) << 32 | int(r[2]):016x}"} for r in stats],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        procs = os.cpu_count() or 1
        try:
            secs = cpu_measure(name, 1, procs)
            line["cpu_baseline"] = {"value": 1.0 / secs, "unit": "frames/s", "cores": procs, "kind": "port",
                                    "sample": f"1 frame pair of {name} (ME+refine+decide+predict) with the numpy "
                                              f"oracle, block rows over {procs} processes"}
        except Exception as exc:  # report, never fake
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=1, help="independent clips per GPU (c4: 64 / world)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process group for the final timing / parity gather (gloo lets ranks share a GPU in tests)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl != "reference" and args.dist_backend == "gloo":
        # test mode: several ranks may share one GPU (no NCCL); the hot path has no collective anyway
        import torch
        local_rank = local_rank % max(1, torch.cuda.device_count())
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group("gloo")
    try:
        return run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""Benchmark: frames/s (and MPix/s) of the per-frame detect+describe hot path.

Workloads (BASELINE.json configs, --config, default 5 = the headline):
  1  640x480, 1 stream, moving objects          2  1280x720, 1 stream, global pan
  3  8 x 1920x1080 streams, one GPU             4  3840x2160, 1 stream, full change every frame
  5  64 x 1920x1080 streams (static / pan / objects), sharded across ranks
Reference defaults t = 55, O = 4; --mode intensity (t_i = 20, the primary
mode), binning or none.  Streams are sharded
contiguously across ranks (strong scaling); a config with fewer streams than
ranks runs one replica per rank (weak scaling).  One step = frame n of every
local stream through the whole path (pyramid -> mask -> score -> NMS/refine ->
describe -> Eq. 1 merge).  Frames come from the CPU scene generator (the same
bytes --impl reference and the parity tests use) and are resident in HBM
before the timed region.

    python bench.py [--config C] [--mode M] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

--impl reference times the reference algorithm on the host cores through the
CPU oracle port (oracle/vf_oracle.c, kind "port"; the reference itself is a
Python package that cannot travel to the GPU box), rank 0 only, on the same
config and bytes.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

TOTAL_STREAMS = 64
W_FR, H_FR = 1920, 1080
PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0  # GB/s, /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="intensity", choices=["intensity", "binning", "none", "temporal"])
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (1: VGA, 2: 720p pan, 3: 8 x 1080p, 4: 4K dense, 5: 64 x 1080p)")
    ap.add_argument("--streams", type=int, default=0, help="override the config's stream count (0 = the config's)")
    ap.add_argument("--gen", default="cpu", choices=["cpu", "cuda"],
                    help="scene generator: cpu = the bytes the reference arm and the parity tests use")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="detect", choices=["detect", "match", "dump", "verify"],
                    help="detect: the headline detect+describe path; match: Hamming radius matching (SURVEY 8(f))")
    ap.add_argument("--match-pairs", type=int, default=8, help="frame pairs per step (match / verify workloads)")
    ap.add_argument("--verify-matches", type=int, default=0,
                    help="verify workload: cap on the match set per pair (first N radius matches; 0 = all)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard(n_total, rank, world):
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return list(range(lo, hi))


def desc_halves(n_streams):
    """Concurrent SAT + describe stream halves of one step (csrc/vf_capi.cu launch_step)."""
    d = max(1, int(os.environ.get("VF_DESC_PAR", "2")))
    return d if n_streams >= d > 1 else 1


def hbm_peak():
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        self._nvml_start()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    # NVML poller (every 2 ms): the timed region can be ~0.1 s, shorter than nvidia-smi's period.
    NVML_BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4}

    def _nvml_start(self):
        self.nv = []
        self.nv_stop = threading.Event()
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = None
            try:
                import torch

                pr = torch.cuda.get_device_properties(torch.cuda.current_device())
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            self.nv_max = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def poll():
                while not self.nv_stop.is_set():
                    try:
                        self.nv.append((time.time(), float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                        int(get_r(h))))
                    except Exception:
                        return
                    time.sleep(0.002)

            self.nv_t = threading.Thread(target=poll, daemon=True)
            self.nv_t.start()
        except Exception:
            self.nv = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def window(self, t0, t1):
        """Keep only samples taken inside [t0, t1] (plus one sampling period)."""
        self.lines = [(t, ln) for t, ln in self.lines if t0 <= t <= t1 + 0.2]
        if self.nv:
            self.nv = [r for r in self.nv if t0 <= r[0] <= t1]

    def __exit__(self, *exc):
        if self.nv is not None:
            self.nv_stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.nv:
            reasons = sorted(k for k, b in self.NVML_BITS.items() if any(r & b for _, _, r in self.nv))
            return {"sm_mhz": statistics.median(c for _, c, _ in self.nv), "sm_max_mhz": self.nv_max,
                    "reasons": reasons, "samples": len(self.nv), "source": "nvml, 2 ms period",
                    "sm_min_mhz": min(c for _, c, _ in self.nv)}
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
# CPU baseline: the oracle port on the host cores (bounded sample)
# ----------------------------------------------------------------------------
def cpu_run(frames_by_stream, mode, threads):
    """frames_by_stream: list of [F, H, W] uint8 arrays.  Returns (frames, seconds)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle
    from paper_1503_06959_b200.pattern import default_pattern

    pat = default_pattern()

    def one(frames):
        p = oracle.OraclePipeline(frames.shape[2], frames.shape[1], pat, mode=mode)
        try:
            for f in frames:
                p.process(f)
        finally:
            p.close()
        return len(frames)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        n = sum(ex.map(one, frames_by_stream))
    return n, time.perf_counter() - t0


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ----------------------------------------------------------------------------
# detect+describe workload: BASELINE.json configs 1..5
# ----------------------------------------------------------------------------
L2_BYTES = 126 << 20          # B200 L2
FLUSH_BYTES = 256 << 20       # written between timed steps when a step's inputs fit in L2
REF_TIME_BUDGET_S = 150.0     # --impl reference: stop timing after this much CPU time (bounded sample)


def config_of(args):
    from paper_1503_06959_b200 import scenes

    cfg = scenes.CONFIGS[args.config]
    n_streams = args.streams if args.streams > 0 else cfg.n_streams
    return cfg, n_streams


def workload_name(args, cfg, n_streams):
    kinds = {"objects": "moving objects", "pan": "global pan + objects", "fresh": "fresh noise every frame",
             "mixed": "static / pan / objects by stream mod 3", "static": "static"}
    return (f"config{args.config}: {n_streams} x {cfg.width}x{cfg.height} uint8 stream{'s' if n_streams > 1 else ''} "
            f"({kinds.get(cfg.kind, cfg.kind)}), mode {args.mode}, t=55, O=4"
            + (", t_i=20" if args.mode == "intensity" else "") + (", 16x16 grid t_h=1" if args.mode == "binning" else ""))


def gen_frames_cpu(cfg, streams, n_frames, device=None, threads=None):
    """[n_frames, S, H, W] uint8 of the given streams from the CPU scene
    generator (the bytes the reference arm and the parity tests use), uploaded
    stream by stream to `device` (None: stays on the host)."""
    from concurrent.futures import ThreadPoolExecutor

    import torch

    from paper_1503_06959_b200 import scenes

    out = torch.empty((n_frames, len(streams), cfg.height, cfg.width), dtype=torch.uint8,
                      device=device if device is not None else "cpu")

    def one(j):
        st = scenes.SceneStream(cfg, streams[j], "cpu")
        buf = torch.stack([st.next_frame() for _ in range(n_frames)])
        out[:, j].copy_(buf, non_blocking=False)
        return j

    nt = threads or host_threads()
    old = torch.get_num_threads()
    torch.set_num_threads(max(1, old // max(1, min(nt, len(streams)))))
    try:
        with ThreadPoolExecutor(max_workers=max(1, min(nt, len(streams)))) as ex:
            list(ex.map(one, range(len(streams))))
    finally:
        torch.set_num_threads(old)
    return out


def gen_frames_cuda(cfg, streams, n_frames, device):
    """[n_frames, S, H, W] uint8 on `device` from the CUDA scene generator (fast; different RNG bytes)."""
    import torch

    from paper_1503_06959_b200 import scenes

    out = torch.empty((n_frames, len(streams), cfg.height, cfg.width), dtype=torch.uint8, device=device)
    for j, s in enumerate(streams):
        st = scenes.SceneStream(cfg, s, device)
        for n in range(n_frames):
            out[n, j] = st.next_frame()
    return out


def gen_frames(streams, n_frames, device):
    """Config-5 frames on the CUDA generator (match / dump workloads)."""
    from paper_1503_06959_b200 import scenes

    return gen_frames_cuda(scenes.CONFIGS[5], streams, n_frames, device)


def layer_areas(W, H, O=4):
    """(rho, top): derived-layer area / WH and top-octave area / WH (pyramid.py:97-125 geometry)."""
    ws, hs = [], []
    ow, oh, iw, ih = W, H, (2 * W) // 3, (2 * H) // 3
    for o in range(O):
        if o:
            ow, oh, iw, ih = ow // 2, oh // 2, iw // 2, ih // 2
        ws += [ow, iw]
        hs += [oh, ih]
    wh = float(W * H)
    rho = sum(w * h for w, h in zip(ws[1:], hs[1:])) / wh
    return rho, ws[2 * (O - 1)] * hs[2 * (O - 1)] / wh


def algorithmic_bytes(W, H, n_frames, cov_sum, k_out, k_prop, k_prev_binning=0.0, O=4):
    """B_alg = sum over frames of W*H*[1 + 2*top + 2*a*(rho - top)]
    + 109*(K_out + K_prop) [+ 16*K_prev in binning mode], with K_out = |D_n| (the
    emitted list, detected + propagated) and K_prop the propagated features read.
    Returns (total, per-kernel shares) -- the shares sum to the total:
      pyramid   reads the frame, writes + re-reads the top octave (IDDM state),
                writes the derived layers within active cells;
      fast      reads the derived layers within active cells;
      describe  writes the detected feature records (109 B);
      propagate reads + writes the propagated records;
      binmask   reads the previous (x, y) pairs (binning mode)."""
    rho, top = layer_areas(W, H, O)
    wh = float(W * H)
    derived = wh * cov_sum * (rho - top)
    k_det = k_out - k_prop
    parts = {
        "pyramid": wh * n_frames * (1 + 2 * top) + derived,
        "fast": derived,
        "describe": 109.0 * k_det,
        "propagate": 218.0 * k_prop,
        "binmask": 16.0 * k_prev_binning,
    }
    return sum(parts.values()), parts


def run_reference(args, rank, world):
    """The reference algorithm on the host cores (oracle/vf_oracle.c, kind
    "port"): the same config, scenes and bytes as the GPU arm (CPU scene
    generator), one frame of each sampled stream per step, one stream per host
    thread.  Streams are sequential in time, so a single-stream config uses one
    core.  Bounded: timing stops after REF_TIME_BUDGET_S."""
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle
    from paper_1503_06959_b200.pattern import default_pattern

    cfg, n_total = config_of(args)
    threads = host_threads()
    n_str = min(n_total, threads)
    streams = list(range(n_str))
    steps = args.warmup + args.steps
    data = gen_frames_cpu(cfg, streams, steps).numpy()       # [F, S, H, W]
    pat = default_pattern()
    W, H = cfg.width, cfg.height
    pipes = [oracle.OraclePipeline(W, H, pat, mode=args.mode) for _ in streams]

    def step(n):
        with ThreadPoolExecutor(max_workers=n_str) as ex:
            list(ex.map(lambda i: pipes[i].process(data[n, i]), range(n_str)))

    for n in range(args.warmup):
        step(n)
    t0 = time.perf_counter()
    done = 0
    for n in range(args.warmup, steps):
        step(n)
        done += 1
        if time.perf_counter() - t0 > REF_TIME_BUDGET_S:
            break
    dt = time.perf_counter() - t0
    for p in pipes:
        p.close()
    frames = n_str * done
    fps = frames / dt
    sample = (f"{n_str} of {n_total} streams x {done} frames (after {args.warmup} warm-up frames), the GPU arm's "
              f"bytes (CPU scene generator); C oracle (oracle/vf_oracle.c), one thread per stream on {cpu_model()}")
    line = {
        "impl": "reference", "metric": "frames/sec (detect+describe)", "value": fps, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": done, "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(done, 1),
        "higher_is_better": True, "scaling": "strong" if n_total > 1 else "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic", "same_config": True,
        "config": {"workload": workload_name(args, cfg, n_total), "sample": sample, "frames": "cpu generator"},
        "mpix_per_sec": fps * W * H / 1e6,
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": n_str, "kind": "port", "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def init_process_group(world, local):
    """NCCL process group (one process per GPU).  At N = 1 a world-size-1 group
    on loopback is created too, so the end-of-run statistics gather is the same
    collective on the measured path at every N."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return "nccl"
    try:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        return "nccl"
    except Exception as e:  # pragma: no cover - reported in the JSON line
        return f"none ({type(e).__name__})"


def launches_per_step(mode, n_streams, width, height):
    # k_pyr_o, k_pyr_i, k_worklist x2 (main + side stream), k_fast, k_nms_list,
    # k_nms_test, k_nms_finish, k_finalize; + k_propagate (mask modes), + k_binmask
    # (binning); the SATs and the describe kernel: early SATs (the default except
    # for intensity-masked batches over 64 MB, vf_capi.cu launch_step) are
    # k_sat_list + k_sat once and k_desc_fused per concurrent describe half, late
    # SATs k_sat + k_desc_fused per half
    env = os.environ.get("VF_SAT_EARLY")
    early = (env != "0") if env is not None else not (mode == "intensity" and width * height * n_streams > (64 << 20))
    halves = desc_halves(n_streams)
    return 9 + (2 + halves if early else 2 * halves) + (1 if mode in ("intensity", "binning") else 0) + (
        1 if mode == "binning" else 0)


def run_detect(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_1503_06959_b200.distributed import gather_stream_history
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    torch.cuda.set_device(local)
    backend = init_process_group(world, local)
    pg = dist.is_available() and dist.is_initialized()
    cfg, n_total = config_of(args)
    W, H = cfg.width, cfg.height
    if n_total >= world:
        streams = shard(n_total, rank, world)
        scaling, ids = "strong", streams
    else:   # fewer streams than GPUs (single-stream configs): independent replicas per rank
        streams = list(range(n_total))
        scaling, ids = "weak", [rank * n_total + s for s in streams]
    S = len(streams)
    Wm, K = args.warmup, args.steps
    e2e_k = 0 if args.no_e2e else max(1, min(args.e2e_steps, K))
    stage_k = max(1, min(10, K))   # eager steps with per-stage CUDA events, after the timed region
    n_frames = Wm + K + stage_k + 2 * e2e_k   # e2e: delta results, then full lists
    dev = torch.device("cuda", local)
    t0g = time.perf_counter()
    if args.gen == "cpu":
        frames = gen_frames_cpu(cfg, streams, n_frames, dev)
    else:
        frames = gen_frames_cuda(cfg, streams, n_frames, dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0g

    eng = FeatureEngine(W, H, PipelineConfig(mask=MaskConfig(mode=args.mode)), n_streams=S)
    hist = torch.zeros((S, Wm + K, 8), dtype=torch.float64, device=dev)
    eng.set_history(hist)
    stream = torch.cuda.current_stream()
    for n in range(Wm):
        eng.process(frames[n])
    torch.cuda.synchronize()

    # ---- timed region: K steps, device-resident inputs ----
    step_bytes = S * W * H
    flush = step_bytes <= L2_BYTES
    flush_buf = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev) if flush else None
    if pg:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(1.0)  # let the samplers start
        tw0 = time.time()
        if flush:
            # a step's inputs fit in L2: write 256 MB between steps, outside the events
            evs = []
            for n in range(Wm, Wm + K):
                flush_buf.fill_(n & 255)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                eng.process(frames[n])
                e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            step_ms = [a.elapsed_time(b) for a, b in evs]
            ms = float(sum(step_ms))
        else:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for n in range(Wm, Wm + K):
                eng.process(frames[n])
            ev1.record(stream)
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
            step_ms = [ms / K] * K
        tw1 = time.time()
    clk.window(tw0, tw1)
    if pg:
        dist.barrier()
    eng.set_history(None)
    # ---- per-stage breakdown: stage_k more steps with CUDA events between the
    # stages (eager launches: the step graph has no stage boundaries) ----
    eng.set_timing(True)
    eng.stage_ms()  # clear
    s0 = Wm + K
    se0 = torch.cuda.Event(enable_timing=True)
    se1 = torch.cuda.Event(enable_timing=True)
    stage_step_ms = 0.0
    for n in range(s0, s0 + stage_k):
        if flush:
            flush_buf.fill_(n & 255)
        se0.record(stream)
        eng.process(frames[n])
        se1.record(stream)
        torch.cuda.synchronize()
        stage_step_ms += se0.elapsed_time(se1)
    stage_step_ms /= stage_k
    stage, n_steps = eng.stage_ms()
    diag = eng.diag()
    eng.set_timing(False)

    # work of the timed frames from the device history (FrameReport rows)
    h = hist.cpu().numpy()
    ht = h[:, Wm:Wm + K]
    k_det_l, k_tot_l = float(ht[:, :, 0].sum()), float(ht[:, :, 2].sum())
    k_prop_l = float(ht[:, :, 1].sum())
    cov_l = float(ht[:, :, 4].sum())
    k_prev_l = float(h[:, Wm - 1:Wm + K - 1, 2].sum()) if (args.mode == "binning" and Wm >= 1) else 0.0
    loc = torch.tensor([ms, k_det_l, k_tot_l, k_prop_l, cov_l, S * K, k_prev_l], dtype=torch.float64, device=dev)
    if world > 1:
        mx = loc.clone()
        dist.all_reduce(mx[:1], op=dist.ReduceOp.MAX)
        sm = loc.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, tot = float(mx[0]), sm.tolist()
    else:
        ms_max, tot = ms, loc.tolist()
    _, k_det, k_tot, k_prop, cov_sum, frames_done, k_prev = tot
    fps = frames_done / (ms_max / 1e3)

    # ---- end-of-run per-stream statistics gather (NCCL all_gather) ----
    t_g = time.perf_counter()
    full = gather_stream_history(hist, ids, [0.0] * Wm + list(step_ms), max(n_total, S * world))
    torch.cuda.synchronize()
    gather_ms = 1e3 * (time.perf_counter() - t_g)
    fs = full[:, Wm:].cpu().numpy()
    stream_stats = {
        "gathered_shape": list(full.shape), "backend": backend, "gather_ms": gather_ms,
        "fields": ["stream", "n_detected", "n_propagated", "n_total", "n_dropped", "coverage", "frame",
                   "n_survivors", "n_candidates", "step_ms"],
        "features_per_frame_by_stream": {"min": float(fs[:, :, 3].mean(1).min()), "max": float(fs[:, :, 3].mean(1).max())},
        "coverage_by_stream": {"min": float(fs[:, :, 5].mean(1).min()), "max": float(fs[:, :, 5].mean(1).max())},
    }

    # ---- e2e: public API with host buffers (H2D of frames + D2H of results inside) ----
    # Two runs of the pipelined API (vf_pipeline_submit / collect, three steps in
    # flight: the H2D of step n+2 is queued while step n+1 computes and step n's
    # result is copied out):
    #   e2e            each step's result as a delta (vf_pipeline_collect_delta):
    #                  the newly detected records + the Eq. 1 keep mask of every
    #                  previous list; the consumer holds list n-1, and
    #                  vf_delta_apply rebuilds list n bit-exactly (tested);
    #   e2e_full_lists every stream's whole merged list copied every step.
    e2e = e2e_full = None
    if e2e_k:
        def e2e_run(first, delta):
            host = frames[first:first + e2e_k].cpu().pin_memory()
            out = eng.alloc_delta(S * max(65536, W * H // 8)) if delta else eng.alloc_host(S * max(65536, W * H // 8))
            collect = eng.collect_delta if delta else eng.collect
            eng.set_delta(delta)
            # untimed warm-up: the GPU kept busy for ~0.2 s so its clocks are up
            # after the host-side preparation above, then the step itself -- buffers
            # and streams on the first step, the CUDA-graph capture of small batches
            # on the second, replays after it
            spin = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
            t_spin = time.perf_counter()
            while time.perf_counter() - t_spin < 0.2:
                for _ in range(20):
                    spin.add_(1)
                torch.cuda.synchronize()
            del spin
            warm = frames[first - 3:first].cpu().pin_memory()
            for wn in (0, 1, 2, 1, 2):
                eng.submit(warm[wn].numpy())
                collect(out)
            torch.cuda.synchronize()
            if pg:
                dist.barrier()
            d2h_total = 0
            t0 = time.perf_counter()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.submit(host[0].numpy())
            if e2e_k > 1:
                eng.submit(host[1].numpy())
            for n in range(e2e_k):
                if n + 2 < e2e_k:
                    eng.submit(host[n + 2].numpy())
                collect(out)
                if delta:
                    d2h_total += int(out["offsets"][S]) * (5 * 8 + 64) + 4 * int(out["keep_offsets"][S]) + 12 * S
                else:
                    d2h_total += int(out["offsets"][S]) * (5 * 8 + 1 + 4 + 64)
            e1.record(stream)
            torch.cuda.synchronize()
            ms_ = max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0))
            tt = torch.tensor([ms_, S * e2e_k, float(d2h_total)], dtype=torch.float64, device=dev)
            if world > 1:
                m2 = tt.clone()
                dist.all_reduce(m2[:1], op=dist.ReduceOp.MAX)
                s2 = tt.clone()
                dist.all_reduce(s2, op=dist.ReduceOp.SUM)
                ms_, fr_, d2h_total = float(m2[0]), float(s2[1]), float(s2[2])
            else:
                fr_ = S * e2e_k
            return {"value": fr_ / (ms_ / 1e3), "unit": "frames/s", "h2d_bytes_per_step": int(S * H * W * world),
                    "d2h_bytes_per_step": int(d2h_total / e2e_k), "steps": e2e_k}

        base = Wm + K + stage_k
        e2e = e2e_run(base, True)
        e2e["api"] = ("vf_pipeline_submit (pinned frames, H2D) + vf_pipeline_collect_delta (every stream's new "
                      "records + Eq. 1 keep mask of its previous list, D2H to pinned; vf_delta_apply rebuilds the "
                      "merged lists bit-exactly), 3 steps in flight")
        e2e_full = e2e_run(base + e2e_k, False)
        e2e_full["api"] = ("vf_pipeline_submit + vf_pipeline_collect (every stream's whole merged list, D2H to "
                           "pinned), 3 steps in flight")

    if rank != 0:
        eng.close()
        if pg:
            dist.destroy_process_group()
        return

    # ---- roofline (live CUDA events inside the timed region) ----
    peak, peak_kind = hbm_peak()
    b_alg, parts = algorithmic_bytes(W, H, frames_done, cov_sum, k_tot, k_prop, k_prev)
    step_ms_avg = ms_max / K
    step_achieved = b_alg / K / (step_ms_avg / 1e3) / 1e9
    rho, top = layer_areas(W, H)
    per_step = 1.0 / max(n_steps, 1)
    # rank-0 shares of the per-kernel bytes (each rank times its own kernels)
    share = S / max(frames_done / K, 1)
    kbytes = {k: v / K * share for k, v in parts.items()}
    overhead = {   # implementation traffic outside SURVEY 8(d)'s algorithmic bytes (per step, this rank)
        "pyramid": W * H * (rho - top) * (S - cov_l / K),           # derived layers written outside active cells
        "sat": 5.0 * 32 * 32 * diag["sat_tiles_built"],           # strip SAT: read 1 B + write 4 B per built pixel
    }
    if stage.get("describe", 0.0) <= 0 and stage.get("sat", 0.0) > 0:
        stage = dict(stage)
        stage["sat+describe"] = stage.pop("sat")
        stage.pop("describe", None)
        kbytes["sat+describe"] = kbytes.pop("describe", 0.0)
        overhead["sat+describe"] = overhead.pop("sat")
    kernels = []
    for k, v in stage.items():
        if v <= 0:
            continue
        ms_k = v * per_step
        ach = kbytes.get(k, 0.0) / (ms_k / 1e3) / 1e9
        row = {"kernel": k, "ms_per_step": ms_k, "share": ms_k / stage_step_ms,
               "algorithmic_bytes": kbytes.get(k, 0.0), "achieved_gbs": ach, "frac": ach / peak}
        if k in overhead:
            row["overhead_bytes"] = overhead[k]
        if k == "propagate":
            row["stream"] = "side stream, overlapped with fast/nms (share = its duration / step)"
        kernels.append(row)
    kernels.sort(key=lambda r: -r["ms_per_step"])
    traffic = None
    tf = ROOT / "profiles" / f"r02_traffic_config{args.config}_{args.mode}.json"
    if tf.exists():
        try:
            tj = json.loads(tf.read_text())
            traffic = tj["dram_bytes_per_step"] * (S / tj.get("streams", S))
        except Exception:
            traffic = None
    roofline = {
        "bound": "hbm", "achieved": step_achieved, "peak": peak, "unit": "GB/s", "frac": step_achieved / peak,
        "traffic": traffic, "kernel": "detect+describe step (all launches of one step)",
        "algorithmic_bytes_per_step": b_alg / K,
        "compulsory_bytes_per_step": (W * H * frames_done + 109.0 * k_tot) / K,
        "bytes_model": "SURVEY.md 8(d): W*H*[1 + 2*top + 2*a*(rho - top)] + 109*(K_out + K_prop), K_out = |D_n|",
        "traffic_source": (f"{tf.relative_to(ROOT)}: sum of ncu dram__bytes_read+write over one step's launches"
                           if traffic is not None else None),
        "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else "fallback",
        "dominant_kernel": kernels[0] if kernels else None,
        "kernels": kernels,
        "kernels_source": (f"per-stage CUDA events on the launch streams over {stage_k} eager steps after the timed "
                           f"region (step {stage_step_ms * 1e3:.1f} us there; the timed steps replay a CUDA graph "
                           f"when a step's frames are <= 64 MB); share = stage time / that step time"),
        "work_last_step": diag,
    }

    # ---- CPU baseline: oracle port on the host cores, bounded sample (rank 0, N = 1) ----
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = host_threads()
        n_str = min(S, threads)
        nf = min(4, Wm + K)  # frame 0 (full detection) + masked frames per sampled stream
        sample = [frames[:nf, j].cpu().numpy() for j in range(n_str)]
        n_cpu, dt = cpu_run(sample, args.mode, threads)
        cpu = {"value": n_cpu / dt, "unit": "frames/s", "cores": n_str, "kind": "port",
               "sample": f"{n_str} streams x {nf} frames (frame 0 full detection + {nf - 1} masked) of the "
                         f"bench workload, C oracle one thread per stream on {cpu_model()}"}

    lat = sorted(step_ms)
    line = {
        "metric": "frames/sec (detect+describe)", "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": K, "warmup": Wm, "ms_per_step": step_ms_avg, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": workload_name(args, cfg, n_total), "config": args.config, "mode": args.mode,
                   "width": W, "height": H, "streams_total": n_total, "streams_per_rank": S,
                   "sharding": "contiguous streams per rank" if scaling == "strong" else "replicas (one stream)",
                   "frames": (f"{args.gen} scene generator" + (" (same bytes as --impl reference and the parity tests)"
                                                               if args.gen == "cpu" else "")),
                   "frame_gen_s": gen_s,
                   "l2": ("inputs fit in L2: 256 MB written between steps, outside the per-step CUDA events"
                          if flush else "inputs larger than L2: every step reads a fresh batch of frames")},
        "mpix_per_sec": fps * W * H / 1e6,
        "latency_ms": {"p50": lat[len(lat) // 2], "p99": lat[min(len(lat) - 1, int(0.99 * len(lat)))],
                       "per": "step (one frame of every local stream)"},
        "features_per_frame": k_tot / max(frames_done, 1),
        "detected_per_frame": (k_tot - k_prop) / max(frames_done, 1),
        "mean_coverage": cov_sum / max(frames_done, 1),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_full_lists": e2e_full,
        "stream_stats": stream_stats,
        "gpu_launches": launches_per_step(args.mode, S, W, H) * K,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    eng.close()
    if pg:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------
# Hamming radius matching workload
# ----------------------------------------------------------------------------
POPC_PEAK_PER_CLK_SM = 15.6   # measured, tools/micro/popc_bench.cu (profiles/r01_popc_peak.txt)
IMMA_PEAK_TOPS = 1112.0       # measured mma.sync m16n8k32 u8, tools/micro/imma_bench.cu (same file)
TC_I8_PEAK_TOPS = 4579.0      # measured tcgen05.mma.kind::i8 M=128 N>=128: 8192 MAC/clk/SM, tools/micro/tc_i8_peak.cu
T_M = 102


def match_descriptors(pairs, device):
    """Packed descriptors of frames 1 and 2 of config-5 streams 0..pairs-1,
    produced by the engine (intensity mode).  Returns [(a, b)] uint8 tensors."""
    import torch

    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    streams = list(range(pairs))
    frames = gen_frames(streams, 3, device)
    eng = FeatureEngine(W_FR, H_FR, PipelineConfig(mask=MaskConfig(mode="intensity")), n_streams=len(streams))
    got = []
    for n in range(3):
        eng.process(frames[n])
        if n >= 1:
            got.append([torch.from_numpy(eng.features_host(s)["desc"]).to(device) for s in range(len(streams))])
    eng.close()
    return [(got[1][s], got[0][s]) for s in range(len(streams))]   # query = frame 2, reference = frame 1


def run_match(args, rank, world, local):
    """One step = radius_match (t_m = 102) of the current frame's features
    against the previous frame's, for every local stream pair (whole 25.7k x
    25.7k all-pairs per stream at 1080p)."""
    import torch
    import torch.distributed as dist

    from paper_1503_06959_b200.matching import radius_match_device

    impl_ref = args.impl == "reference"
    if impl_ref and rank != 0:
        return
    if not impl_ref:
        torch.cuda.set_device(local)
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if impl_ref:
        # same inputs, produced on the host by the oracle (the reference arm uses no GPU code)
        from oracle import oracle
        from paper_1503_06959_b200 import scenes
        from paper_1503_06959_b200.pattern import default_pattern

        pairs = []
        for s_ in range(args.match_pairs):
            fr = scenes.generate(scenes.CONFIGS[5], 3, streams=[s_])[0].numpy()
            seq = oracle.run_sequence(list(fr), default_pattern(), mode="intensity")
            pairs.append((torch.from_numpy(seq[2].desc), torch.from_numpy(seq[1].desc)))
    else:
        dev = torch.device("cuda", local)
        mine = shard(args.match_pairs, rank, world)
        pairs_all = match_descriptors(args.match_pairs, dev)
        pairs = [pairs_all[i] for i in mine]
    n_pairs_step = float(sum(a.shape[0] * b.shape[0] for a, b in pairs))
    cfg = {"workload": f"match: radius_match t_m={T_M} of frame-2 vs frame-1 packed 512-bit descriptors of "
                       f"{args.match_pairs} config-5 1080p streams (intensity mode)",
           "pairs_per_step": n_pairs_step * (world if not impl_ref else 1),
           "descriptors_per_frame": float(np.mean([a.shape[0] for a, _ in pairs]))}
    if impl_ref:
        from concurrent.futures import ThreadPoolExecutor

        from oracle import oracle

        threads = host_threads()
        host = [(a.cpu().numpy(), b.cpu().numpy()) for a, b in pairs]
        rows = 256   # bounded sample per step: 256 query rows of every pair
        jobs = [(a[i:i + 16], b) for a, b in host for i in range(0, rows, 16)]

        def step():
            with ThreadPoolExecutor(max_workers=threads) as ex:
                return sum(ex.map(lambda j: len(oracle.radius_match(j[0], j[1], T_M)[0]), jobs))

        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        dt = (time.perf_counter() - t0) / args.steps
        pps = sum(j[0].shape[0] * j[1].shape[0] for j in jobs) / dt
        line = {"impl": "reference", "metric": "descriptor pairs/s (Hamming radius match)", "value": pps,
                "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "u32 (popcount)", "data": "synthetic", "config": cfg,
                "cpu_baseline": {"value": pps, "unit": "pairs/s", "cores": threads, "kind": "port",
                                 "sample": f"{rows} query rows x all reference rows of each of {len(host)} pairs per "
                                           f"step; C oracle (LUT popcount, matching.py:47-66) on {cpu_model()}"},
                "e2e": {"value": pps, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > L2 (126 MB): written between steps
    n_match = 0

    def step():
        nonlocal n_match
        n = 0
        for a, b in pairs:
            qi, _, _ = radius_match_device(a, b, T_M)
            n += qi.numel()
        n_match = n

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    from paper_1503_06959_b200 import _native

    L = _native.lib()
    kern_ms = ctypes.c_double(0.0)
    _native.check(L.vf_match_timing(1, None))
    ms = 0.0
    with ClockSampler(local) as clk:
        time.sleep(1.0)
        tw0 = time.time()
        for _ in range(args.steps):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()      # radius_match synchronizes (match count) -- inside the events
            e1.record(stream)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        tw1 = time.time()
    clk.window(tw0, tw1)
    _native.check(L.vf_match_timing(0, ctypes.byref(kern_ms)))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t[0])
    pps = n_pairs_step * world * args.steps / (ms_max / 1e3)
    # distance kernel of the timed radius matches (operand images + k_radius_tc,
    # CUDA events on the call's stream inside vf_radius_match)
    kms = kern_ms.value / args.steps
    # tensor-core path: q.r of 512 0/1 bytes per pair (2 x 512 int8 ops per pair)
    ops = 2.0 * 512 * n_pairs_step
    peak = TC_I8_PEAK_TOPS
    ach = ops / (kms / 1e3) / 1e12
    # e2e: host packed descriptors (pinned) -> H2D -> radius match -> D2H of the matches
    host = [(a.cpu().pin_memory(), b.cpu().pin_memory()) for a, b in pairs]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h2d = d2h = 0
    for a, b in host:
        ad, bd = a.to(dev, non_blocking=True), b.to(dev, non_blocking=True)
        qi, ri, d = radius_match_device(ad, bd, T_M)
        out = torch.stack([qi, ri, d]).cpu()
        h2d += a.numel() + b.numel()
        d2h += out.numel() * 4
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if rank == 0:
        line = {"metric": "descriptor pairs/s (Hamming radius match)", "value": pps, "unit": "pairs/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32 (popcount)",
                "data": "synthetic", "config": dict(cfg, l2="256 MB buffer written between timed steps (outside "
                                                         "the events)", matches_per_step=n_match * world),
                "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TOPS (int8)",
                             "frac": ach / peak, "traffic": None,
                             "kernel": "k_tc_images + k_radius_tc (tcgen05.mma.kind::i8, TMEM accumulators; live CUDA "
                                       "events around the distance kernel of every timed radius match)",
                             "peak_source": "measured tcgen05.mma.kind::i8 M=128 N=128 issue rate, 8192 MAC/clk/SM "
                                            "(tools/micro/tc_i8_peak.cu, profiles/r01e_tc_i8_peak.txt)",
                             "kernel_ms_per_step": kms},
                "e2e": {"value": n_pairs_step / e2e_s, "unit": "pairs/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "api": "pinned packed descriptors -> radius_match_device -> "
                                                          "matches to host"},
                "gpu_launches": args.steps * len(pairs) * 3, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def verify_sets(pairs, n_max, device, impl_ref):
    """(src, dst) match coordinates of radius_match(frame 2, frame 1, t_m) for
    config-5 streams 0..pairs-1 (CPU-generated frames in both arms): the
    count_mpr input between consecutive frames (matching.py:209-220).  Each
    set is the first n_max matches in np.nonzero order (all if n_max <= 0).
    Built on the GPU (engine + radius match) for our arm, by the oracle on the
    host for the reference arm."""
    import torch

    from paper_1503_06959_b200 import scenes
    from paper_1503_06959_b200.pattern import default_pattern

    sets = []
    if impl_ref:
        from oracle import oracle

        for s_ in range(pairs):
            fr = scenes.generate(scenes.CONFIGS[5], 3, streams=[s_])[0].numpy()
            seq = oracle.run_sequence(list(fr), default_pattern(), mode="intensity")
            qs, rs, r0 = [], [], 0
            while r0 < len(seq[2].desc) and (n_max <= 0 or sum(map(len, qs)) < n_max):   # leading rows only
                a, b, _ = oracle.radius_match(seq[2].desc[r0:r0 + 256], seq[1].desc, T_M)
                qs.append(a + r0)
                rs.append(b)
                r0 += 256
            qi, ri = np.concatenate(qs), np.concatenate(rs)
            if n_max > 0:
                qi, ri = qi[:n_max], ri[:n_max]
            sets.append((np.stack([seq[2].x[qi], seq[2].y[qi]], 1), np.stack([seq[1].x[ri], seq[1].y[ri]], 1)))
        return sets
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.matching import radius_match_device
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    # frames drawn on the CPU generator, as the reference arm's: both arms verify identical match sets
    frames = scenes.generate(scenes.CONFIGS[5], 3, streams=range(pairs)).permute(1, 0, 2, 3).contiguous().to(device)
    eng = FeatureEngine(W_FR, H_FR, PipelineConfig(mask=MaskConfig(mode="intensity")), n_streams=pairs)
    got = []
    for n in range(3):
        eng.process(frames[n])
        if n >= 1:
            got.append([eng.features_host(s) for s in range(pairs)])
    eng.close()
    for s_ in range(pairs):
        a, b = got[1][s_], got[0][s_]
        qi, ri, _ = radius_match_device(torch.from_numpy(a["desc"]).to(device), torch.from_numpy(b["desc"]).to(device),
                                        T_M)
        if n_max > 0:
            qi, ri = qi[:n_max], ri[:n_max]
        qi, ri = qi.cpu().numpy(), ri.cpu().numpy()
        sets.append((np.stack([a["x"][qi], a["y"][qi]], 1), np.stack([b["x"][ri], b["y"][ri]], 1)))
    return sets


def run_verify(args, rank, world, local):
    """One step = ransac_homography (1000 iterations, tol 3 px, seed 0) of
    every local pair's match set: count_mpr's verification between frame 2
    and frame 1 of config-5 1080p streams."""
    import torch
    import torch.distributed as dist

    iters, tol = 1000, 3.0
    impl_ref = args.impl == "reference"
    if impl_ref and rank != 0:
        return
    if not impl_ref:
        torch.cuda.set_device(local)
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local) if not impl_ref else None
    mine = shard(args.match_pairs, rank, world) if not impl_ref else list(range(args.match_pairs))
    sets_all = verify_sets(args.match_pairs, args.verify_matches, dev, impl_ref)
    sets = [sets_all[i] for i in mine]
    n_pts = [len(s) for s, _ in sets]
    cfg = {"workload": f"verify: ransac_homography ({iters} iterations, tol {tol} px, seed 0) of the radius "
                       f"matches (t_m={T_M}, {'first ' + str(args.verify_matches) if args.verify_matches > 0 else 'all'}) between frames 2 and 1 of "
                       f"{args.match_pairs} config-5 1080p streams (intensity mode)",
           "match_sets_per_step": len(sets) * (world if not impl_ref else 1),
           "matches_per_set": float(np.mean(n_pts)), "iterations": iters}
    metric = "match sets verified/s (ransac_homography, 1000 iterations)"
    if impl_ref:
        from concurrent.futures import ThreadPoolExecutor

        from oracle import oracle

        threads = host_threads()
        s_iters = 40    # bounded sample: 40 of the 1000 iterations per set, scaled (the refit is O(n))

        def one(j):
            src, dst = sets[j]
            return oracle.ransac_homography(src, dst, s_iters, tol, 0)

        def step():
            with ThreadPoolExecutor(max_workers=threads) as ex:
                return list(ex.map(one, range(len(sets))))

        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        dt = (time.perf_counter() - t0) / args.steps * (iters / s_iters)
        v = len(sets) / dt
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "sets/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
                "cpu_baseline": {"value": v, "unit": "sets/s", "cores": min(threads, len(sets)), "kind": "port",
                                 "sample": f"{s_iters} of {iters} RANSAC iterations of each of {len(sets)} sets per "
                                           f"step, time scaled x{iters // s_iters}; C oracle (normalized DLT via "
                                           f"Jacobi SVD, matching.py:97-192), one set per thread on {cpu_model()}"},
                "e2e": {"value": v, "unit": "sets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    from paper_1503_06959_b200.matching import ransac_homography_batch, ransac_homography_device

    off = np.zeros(len(sets) + 1, np.int64)
    off[1:] = np.cumsum(n_pts)
    src = torch.from_numpy(np.concatenate([s for s, _ in sets])).to(dev)
    dst = torch.from_numpy(np.concatenate([d for _, d in sets])).to(dev)
    stream = torch.cuda.current_stream()

    def step():
        return ransac_homography_device(src, dst, off, iters, tol, 0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = 0.0
    with ClockSampler(local) as clk:
        time.sleep(1.0)
        tw0 = time.time()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            _, _, cnt = step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        tw1 = time.time()
    clk.window(tw0, tw1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t[0])
    v = len(sets) * world * args.steps / (ms_max / 1e3)
    evals = float(sum(n_pts)) * iters
    # e2e: host match coordinates -> H2D -> RANSAC -> (H, counts, inlier masks) to host, per step
    host = [(s.copy(), d.copy()) for s, d in sets]
    e2e_k = max(1, min(args.e2e_steps, args.steps))
    ransac_homography_batch(host, iters, tol, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_k):
        res = ransac_homography_batch(host, iters, tol, 0)
    e2e_s = (time.perf_counter() - t0) / e2e_k
    h2d = int(2 * 16 * sum(n_pts) + 8 * (len(sets) + 1))
    d2h = int(len(sets) * (72 + 4) + sum(n_pts))
    if rank == 0:
        line = {"metric": metric, "value": v, "unit": "sets/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(cfg, l2=f"inputs ({32 * sum(n_pts) / 1e6:.1f} MB of coordinates) stay L2-resident "
                                       "by design: every set is re-read by 1000 hypotheses",
                               mpr=[len(r[1]) for r in res][:8]),
                "roofline": verify_roofline(evals * world * args.steps / (ms_max / 1e3) / 1e9),
                "e2e": {"value": len(sets) / e2e_s, "unit": "sets/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "api": "host (src, dst) arrays -> ransac_homography_batch -> "
                                                          "(H, inlier lists) on the host"},
                "gpu_launches": args.steps * 11, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def verify_roofline(achieved_g):
    """k_rs_score is fp64-pipe bound (16.5 fp64 instructions per
    hypothesis-match evaluation); frac = the fp64 pipe's active fraction from
    the committed ncu capture (profiles/r01d_verify_score.json), peak = the
    evaluation rate at a fully busy pipe implied by it."""
    prof = ROOT / "profiles" / "r01d_verify_score.json"
    frac = None
    if prof.exists():
        frac = json.loads(prof.read_text()).get("sm__pipe_fp64_cycles_active_pct", None)
        frac = frac / 100.0 if frac else None
    return {"bound": "fp64", "achieved": achieved_g, "peak": achieved_g / frac if frac else None,
            "unit": "G hypothesis-match evaluations/s", "frac": frac,
            "traffic": 42758912 + 51456 if prof.exists() else None,
            "kernel": "k_rs_score (92% of the call; whole-step rate from live CUDA events)",
            "peak_source": "fp64 pipe utilization of k_rs_score, ncu --set full (profiles/r01d_verify_score.json)"}


def run_dump(args):
    """Feature-dump formatting (report.py:96-113): the
    features of one config-5 step (all streams, one frame) as dump_features
    text, native formatter vs the reference's Python f-string loop."""
    import torch

    from oracle import oracle
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.report import format_features
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    streams = list(range(min(args.streams or TOTAL_STREAMS, 64)))
    frames = gen_frames(streams, 3, torch.device("cuda", 0))
    eng = FeatureEngine(W_FR, H_FR, PipelineConfig(mask=MaskConfig(mode="intensity")), n_streams=len(streams))
    for n in range(3):
        eng.process(frames[n])
    soas = [eng.features_host(s) for s in range(len(streams))]
    eng.close()
    n_feat = sum(len(f["x"]) for f in soas)
    threads = host_threads()
    if args.impl == "reference":
        sample = soas[:2]
        n_s = sum(len(f["x"]) for f in sample)
        t0 = time.perf_counter()
        for _ in range(max(1, args.steps)):
            for f in sample:
                oracle.dump_lines(f["x"], f["y"], f["sigma"], f["theta"], f["origin"], f["desc"])
        dt = (time.perf_counter() - t0) / max(1, args.steps)
        v = n_s / dt
        print(json.dumps({"impl": "reference", "metric": "features/s (feature dump text)", "value": v,
                          "unit": "features/s", "n_gpus": 1, "steps": args.steps, "warmup": 0,
                          "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                          "dtype": "text", "data": "synthetic",
                          "config": {"workload": "dump: report.dump_features lines of config-5 features",
                                     "features": n_s},
                          "cpu_baseline": {"value": v, "unit": "features/s", "cores": 1, "kind": "port",
                                           "sample": f"{len(sample)} streams x 1 frame ({n_s} features), Python "
                                                     "f-string loop of report.py:102-113 (oracle.dump_lines)"},
                          "e2e": {"value": v, "unit": "features/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    for _ in range(args.warmup):
        for f in soas:
            format_features(f)
    t0 = time.perf_counter()
    nbytes = 0
    for _ in range(args.steps):
        for f in soas:
            nbytes += len(format_features(f))
    dt = (time.perf_counter() - t0) / args.steps
    print(json.dumps({"metric": "features/s (feature dump text)", "value": n_feat / dt, "unit": "features/s",
                      "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
                      "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "text",
                      "data": "synthetic",
                      "config": {"workload": f"dump: report.dump_features lines of {len(streams)} config-5 streams "
                                             f"(one frame each)", "features": n_feat,
                                 "text_mb_per_step": nbytes / args.steps / 1e6},
                      "roofline": {"bound": "host", "achieved": nbytes / args.steps / dt / 1e9, "peak": None,
                                   "unit": "GB/s of text", "frac": None, "traffic": None,
                                   "kernel": f"vf_format_features (C++, {threads} host threads)"},
                      "gpu_launches": 0}), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.workload == "dump":
        if rank == 0:
            run_dump(args)
        return
    if args.workload == "match":
        run_match(args, rank, world, local)
        return
    if args.workload == "verify":
        run_verify(args, rank, world, local)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_detect(args, rank, world, local)


if __name__ == "__main__":
    main()

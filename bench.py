#!/usr/bin/env python
"""Benchmark: 4-direction 5x5 Sobel on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload 8k|1080p-batch|32k-bands] [--contract sr|u8|sr32]

One "step" = one pass of the hot path over one synthetic image (or batch):
the fused sm_100a kernel over an input already resident in HBM; the K timed
steps are captured after the warm-up as one CUDA graph and replayed once
(--no-graph: a Python launch loop).  Default
workload is BASELINE config C3, 7680x4320 uint8 (the north-star roofline
case); at N>1 every rank processes its own frame (weak scaling, no
communication: the batch-split sharding of SURVEY.md section 8e).

Prints ONE JSON line (rank 0).  `value` is whole-job Gpixel/s (input pixels,
metrics.hpp:176 convention) timed with CUDA events on the launching stream,
max over ranks; `e2e` is the same metric through the C ABI host-buffer entry
(sobel5_run_host) with pinned host buffers, copies inside the timed region;
`roofline` is algorithmic bytes per launch / launch time vs the measured HBM
copy bandwidth; `cpu_baseline` is the reference's own run_stream compiled from
its headers (oracle/_ref) timed on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpixel/s and achieved HBM GB/s (% of peak) for 4-dir 5x5 Sobel, 1/2/4/8 B200"
UNIT = "Gpixel/s"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback
OUT_BYTES = {"sr": 24, "sr32": 20, "u8": 1}  # per output pixel
CONTRACT_PLANES = {"sr": ("gx", "gy", "gd", "gdt", "g"), "sr32": ("gx", "gy", "gd", "gdt", "g32"),
                   "u8": ("u8",)}
WORKLOADS = {
    "8k": dict(w=7680, h=4320, frames=1, name="7680x4320 uint8 single image (BASELINE C3)"),
    "4k": dict(w=3840, h=2160, frames=1, name="3840x2160 uint8 single image (BASELINE C2)"),
    "1080p-batch": dict(w=1920, h=1080, frames=256,
                        name="batch of 256 1920x1080 uint8 frames split across ranks (C4)"),
    "32k-bands": dict(w=32768, h=32768, frames=1,
                      name="32768x32768 uint8 single image row-band partitioned across ranks "
                           "with 2-row halos (C5)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: 8k (C3) at N=1, 32k-bands (C5, one image row-band "
                         "partitioned over the ranks) at N>1")
    ap.add_argument("--contract", default="sr", choices=sorted(OUT_BYTES))
    ap.add_argument("--prefetch", type=int, default=1)
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl", "gloo"],
                    help="32k-bands halo transport")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the K steps as a Python launch loop instead of one CUDA graph")
    ap.add_argument("--share-gpu", action="store_true",
                    help="testing only: every rank uses cuda:0 and gloo (exercises the N>1 "
                         "code path on a one-GPU box; numbers are not scaling numbers)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="budget of CPU work for the cpu_baseline sample")
    ap.add_argument("--no-cpu-matrix", action="store_true",
                    help="skip the BASELINE.md section 2 CPU matrix (C1-C3 x lanes x workers)")
    a = ap.parse_args()
    if a.workload is None:
        a.workload = "32k-bands" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "8k"
    return a


def base_config(a, world: int) -> dict:
    """The workload description both arms print (identical dicts)."""
    wl = WORKLOADS[a.workload]
    frames = wl["frames"] if wl["frames"] == 1 else max(1, wl["frames"] // world)
    return {"workload": wl["name"], "frames_per_rank": frames,
            "contract": a.contract + " (" + "+".join(CONTRACT_PLANES[a.contract]) + ")",
            "prefetch": bool(a.prefetch),
            "parallelism": (f"row-bands x{world} ({a.transport} halos)"
                            if a.workload == "32k-bands" else f"batch-split x{world}"),
            # L2 policy of the GPU timing (126 MB L2): no L2 flush; every step
            # reads an input larger than L2 or rotates inputs over > 2x L2, and
            # writes outputs far larger than L2
            "l2": ("inputs larger than L2: each rank's 32768-wide band (>= 128 MB) read "
                   "once per step, outputs >= 3.2 GB per step" if a.workload == "32k-bands"
                   else "inputs rotated over >= 2 x L2 of frames (no L2 flush)")}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return FALLBACK_HBM_GBS, "fallback", {}


# ---- clocks sampling (nvml) during the timed region --------------------------------


class ClockSampler:
    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000010: "sync_boost", 0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown", 0x0000000000000080: "hw_power_brake_slowdown",
        0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv, self.err = None, str(e)

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mask = fn(self.h)
        for bit, name in self.REASONS.items():
            if mask & bit and name != "gpu_idle":
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.005)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self.nv:
            self._stop.set()
            self._t.join()
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---- CPU reference arm ----------------------------------------------------------------


def cpu_reference(w, h, frames, seconds, max_iters=None):
    """The reference's run_stream (pipeline.hpp:474) from its own headers,
    lanes 256, prefetch on, one worker per host core, timed with the
    reference's measure() (metrics.hpp:142-179).  Falls back to the C oracle
    port when the compiled reference is absent."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    cores = os.cpu_count() or 1
    rows = h if w * h <= 40_000_000 else max(5, int(40_000_000 // w))  # 32K: a band of rows
    unit = "frame" if rows == h else f"{rows}-row band of the frame"
    if pyoracle.ref_available():
        R = pyoracle.Reference()
        img = R.synth_random(w, rows, 1)
        t0 = time.perf_counter()
        mean1, _ = R.measure_run_stream(img, lanes=256, prefetch=True, workers=cores, iters=1)
        first = time.perf_counter() - t0
        iters = max(1, min(30, int(seconds / max(mean1, 1e-6))))
        if max_iters:
            iters = min(iters, max_iters)
        mean, sd = R.measure_run_stream(img, lanes=256, prefetch=True, workers=cores,
                                        iters=iters)
        kind = "reference"
        sample = (f"{iters} timed + 1 warm-up reference run_stream calls (lanes 256, prefetch on, "
                  f"workers {cores}) on one {w}x{rows} synth_random {unit}; first call "
                  f"{first:.2f}s")
        cores_used = cores
    else:  # oracle port, single thread
        O = pyoracle.Oracle()
        img = O.synth_random(w, rows, 1)
        t0 = time.perf_counter()
        O.run_stream(img)
        mean = time.perf_counter() - t0
        sd, kind, cores_used = 0.0, "port", 1
        sample = f"1 oracle-port run_stream call on one {w}x{rows} {unit} (reference not built)"
    gpx = w * rows / mean / 1e9
    return {"value": gpx, "unit": UNIT, "cores": cores_used, "kind": kind, "sample": sample,
            "mean_s_per_frame": mean, "stddev_s": sd,
            "note": f"per-frame rate; a {frames}-frame workload scales linearly"}


def run_reference_arm(a):
    """The reference's own CPU implementation of the path (run_stream from its
    headers, oracle/_ref; the C oracle port where it is absent) on this
    host's cores, timed with the reference's measure(): W warm-up runs then
    exactly K timed steps, each step a bounded sample of the workload --
    whole frames (C3: one 8K frame; C4: frames of the batch) or, for the
    32K image, a band of its rows -- sized to ~0.5 s.  Rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    wl = WORKLOADS[a.workload]
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    cores = os.cpu_count() or 1
    w, h = wl["w"], wl["h"]
    have_ref = pyoracle.ref_available()
    G = pyoracle.Reference() if have_ref else pyoracle.Oracle()
    # sample: rows of the workload's image (a whole frame where it fits)
    rows = h
    if w * h > 40_000_000:  # the 32K image: a band of rows
        rows = max(5, min(h, int(40_000_000 // w)))
    img = G.synth_random(w, rows, 1)

    def run_once():
        if have_ref:
            return G.measure_run_stream(img, lanes=256, prefetch=True, workers=cores, iters=1)[0]
        t0 = time.perf_counter()
        G.run_stream(img)
        return time.perf_counter() - t0

    for _ in range(a.warmup):
        run_once()
    if have_ref:  # measure() adds one untimed call of its own
        mean, sd = G.measure_run_stream(img, lanes=256, prefetch=True, workers=cores,
                                        iters=a.steps)
        kind, cores_used = "reference", cores
    else:
        ts = [run_once() for _ in range(a.steps)]
        mean, sd = statistics.mean(ts), statistics.pstdev(ts)
        kind, cores_used = "port", 1
    gpx = w * rows / mean / 1e9
    unit = "frame" if rows == h else f"band of {rows} rows"
    sample = (f"each step: one reference run_stream call (lanes 256, prefetch on, workers "
              f"{cores_used}) on a {w}x{rows} synth_random {unit} of the workload; "
              f"{a.warmup} warm-up + {a.steps} timed steps")
    line = {"metric": METRIC, "value": gpx, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": mean * 1e3,
            "higher_is_better": True, "scaling": "strong" if a.workload == "32k-bands" else "weak",
            "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (synth_random seed 1)",
            "config": base_config(a, world),
            "stddev_s": sd,
            "cpu_baseline": {"value": gpx, "unit": UNIT, "cores": cores_used, "kind": kind,
                             "sample": sample, "host": host_cpu()},
            "e2e": {"value": gpx, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def host_cpu() -> dict:
    """nproc and the lscpu model of this host (for the CPU numbers)."""
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def cpu_matrix(budget_s: float = 60.0) -> dict:
    """BASELINE.md section 2's CPU matrix: the reference's run_stream at
    lanes 32 / 256 x workers 1 / nproc and its single-thread sobel5_4d
    oracle, on C1-C3, each through the reference's measure() (1 warm-up + 2
    timed calls), rows in its BenchReport CSV schema (metrics.hpp:129-139)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    if not pyoracle.ref_available():
        return {"skipped": "oracle/_ref not built"}
    R = pyoracle.Reference()
    cores = os.cpu_count() or 1
    rows, t_start = [], time.perf_counter()
    for (w, h) in ((1920, 1080), (3840, 2160), (7680, 4320)):
        img = R.synth_random(w, h, 1)
        for which, lanes, workers in (("fast", 32, 1), ("fast", 256, 1), ("fast", 32, cores),
                                      ("fast", 256, cores), ("oracle", 0, 1)):
            if rows and time.perf_counter() - t_start > budget_s:
                break
            _, row = R.measure_csv(img, which, lanes or 32, True, workers, 2)
            rows.append({"lanes": lanes or None, "workers": workers, "csv": row})
    return {"csv_header": "label,width,height,iters,mean_s,stddev_s,mps,mps_per_core",
            "rows": rows, "host": host_cpu(),
            "note": "reference headers compiled -O3 -DNDEBUG (oracle/_ref); fast-5x5 = "
                    "run_stream prefetch on, oracle-5x5 = sobel5_4d; mps = megapixels/s"}


# ---- our arm ------------------------------------------------------------------------------


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference_arm(a)

    rank, world, local = dist_env()
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2305_00515_b200 import _abi, api
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    if a.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if a.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    _abi.load()

    wl = WORKLOADS[a.workload]
    w, h = wl["w"], wl["h"]
    frames = wl["frames"]
    if frames > 1:  # batch split across ranks, no communication (C4)
        frames = max(1, frames // world)
    ow, oh = w - 4, h - 4
    planes_names = CONTRACT_PLANES[a.contract]
    taps = api.make_stream_taps()
    taps_default = True  # (1, 2, 6, 4): the packed kernel (sobel5_packed.cuh)
    stream = torch.cuda.current_stream(dev)
    s_ptr = stream.cuda_stream

    scaling = "weak"
    if a.workload == "32k-bands":
        # C5: one 32768^2 image row-band partitioned over the ranks (strong
        # scaling); halos from the neighbours via peer-mapped buffers read
        # inside the kernel (default) or NCCL send/recv (--transport nccl)
        from paper_2305_00515_b200.bands import RowBandPartition, plan_bands
        scaling = "strong"
        plan = plan_bands(w, h, world, rank)
        body, pitch = api.alloc_input(w, plan.body_rows, dev)
        api.synth_random_device(body, pitch, w, plan.body_rows, seed=1, row_offset=plan.r0,
                                stream=s_ptr)
        torch.cuda.synchronize()
        part = RowBandPartition(plan, body, pitch, transport=a.transport)
        out, op = api.alloc_planes(ow, plan.out_rows, planes_names, dev)
        n_in, in_bytes = 1, w * plan.body_rows
        px_job = w * h
        rank_in_px, rank_out_px = w * plan.body_rows, ow * plan.out_rows

        def step(i, sp=s_ptr):
            part.run(taps, out, op, a.prefetch, stream=sp)
    else:
        # Inputs: rotate over enough frames that the input set exceeds L2
        # (126 MB); the outputs alone (24 B/px) are 6x L2 at 8K.
        in_bytes = w * h * frames
        n_in = max(2, int(np.ceil(2 * 126e6 / in_bytes)))
        n_in = min(n_in, 8)
        ins = []
        for i in range(n_in):
            d, pitch = api.alloc_input(w, h, dev, frames=frames)
            for f in range(frames):
                sub = d[f] if frames > 1 else d
                api.synth_random_device(sub, pitch, w, h, seed=1 + (rank * frames + f) + i * 1000,
                                        stream=s_ptr)
            ins.append(d)
        out, op = api.alloc_planes(ow, oh, planes_names, dev, frames=frames)
        px_job = w * h * frames * world
        rank_in_px, rank_out_px = w * h * frames, ow * oh * frames

        def step(i, sp=s_ptr):
            d = ins[i % n_in]
            if frames > 1:
                api.launch_batch(d, pitch, h * pitch, w, h, frames, taps, a.prefetch, out, op,
                                 oh * op, stream=sp)
            else:
                api.launch(d, pitch, w, h, taps, a.prefetch, out, op, stream=sp)
    torch.cuda.synchronize()

    for i in range(a.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # The K timed steps run as ONE CUDA graph (captured after the warm-up):
    # the device time of the steps without Python's per-launch host cost
    # between them, as a production loop over frames would issue them.
    # Host-synchronising transports (nccl / gloo halos) run as a plain loop.
    # (the peer transport orders ranks with per-step flag values, which a
    # graph replay would freeze at their capture-time values)
    use_graph = not a.no_graph and not (a.workload == "32k-bands" and world > 1)
    run_stream_obj = stream  # CUDAGraph.replay() launches on the current stream
    if use_graph:
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        n0 = api.launch_count()
        with torch.cuda.graph(graph, stream=gs):
            for i in range(a.steps):
                step(i, gs.cuda_stream)
        launches_per_replay = api.launch_count() - n0
        graph.replay()  # one untimed replay (graph upload); replays run on `stream`
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    launches0 = api.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    e0.record(run_stream_obj)
    if use_graph:
        graph.replay()
    else:
        for i in range(a.steps):
            step(i)
    e1.record(run_stream_obj)
    torch.cuda.synchronize()
    clocks.stop()
    launches = launches_per_replay if use_graph else api.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cpu" if a.share_gpu else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    torch.cuda.synchronize()
    ms_step = ms / a.steps
    value = px_job / (ms_step * 1e-3) / 1e9
    # spread (median and mean +- stddev): 4 more timed replays of
    # the same graph on rank 0's device; the headline stays the first one
    rep_ms = [ms_step]
    if use_graph and world == 1:
        for _ in range(4):
            e0.record(run_stream_obj)
            graph.replay()
            e1.record(run_stream_obj)
            torch.cuda.synchronize()
            rep_ms.append(e0.elapsed_time(e1) / a.steps)
    spread = {"replays": len(rep_ms), "median_ms_per_step": float(np.median(rep_ms)),
              "mean_ms_per_step": float(np.mean(rep_ms)),
              "stddev_ms_per_step": float(np.std(rep_ms))}

    hbm_peak, peak_kind, peaks = measured_peaks()
    alg_bytes = rank_in_px + rank_out_px * OUT_BYTES[a.contract]  # per rank, per launch set
    achieved = alg_bytes / (ms_step * 1e-3) / 1e9
    # steady-state ncu numbers per launch (tools/traffic.sh + tools/traffic.py):
    # DRAM bytes and warp-instructions of the same kernel at the same size
    traffic, traffic_ratio, prof = None, None, {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                prof = json.load(f)
            t = prof.get(f"{a.workload}/{a.contract}")
            if isinstance(t, dict) and frames == 1 and world == 1:
                traffic = t["traffic"]
                traffic_ratio = t["traffic"] / alg_bytes
        except Exception:
            traffic, prof = None, {}

    def issue_frac(key, us):
        """Issue-rate roofline of an issue-bound kernel: its ncu warp-instruction
        count per launch over what 4 SMSPs x 148 SMs issue at the run's median SM
        clock in the measured time (1.0 = one instruction per SMSP per cycle)."""
        t = prof.get(key)
        mhz = clocks.summary().get("sm_mhz") or 1965.0
        if not isinstance(t, dict) or not us:
            return None
        return {"frac": t["inst_per_launch"] / (4 * 148 * mhz * us),
                "inst_per_launch": t["inst_per_launch"],
                "thread_inst_per_px": t["inst_per_launch"] * 32 / (ow * oh),
                "source": "profiles/traffic.json (ncu smsp__inst_executed.sum)"}

    # ---- variants (same workload, other output contracts / paths) ----
    # Each is timed like the headline (CUDA events around n launches on the
    # launching stream, inputs rotated over > L2); bytes are algorithmic
    # (input read once + outputs written once).
    variants = {}
    if rank == 0 and frames == 1 and a.workload != "32k-bands":
        scratch = api.alloc_scratch(1, dev, out_h=h, pitch=api.round_up(w, 32))

        def variant(name, planes_names_v, out_w_v, out_h_v, out_bytes_px, call, passes=1):
            # timed like the headline: 50 calls captured in one CUDA graph
            vo, vp = api.alloc_planes(out_w_v, out_h_v, planes_names_v, dev)
            for i in range(5):
                call(ins[i % n_in], vo, vp, s_ptr)
            torch.cuda.synchronize()
            n = 50
            vs = torch.cuda.Stream(dev)
            vs.wait_stream(stream)
            vg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(vg, stream=vs):
                for i in range(n):
                    call(ins[i % n_in], vo, vp, vs.cuda_stream)
            vg.replay()
            torch.cuda.synchronize()
            v0, v1 = torch.cuda.Event(True), torch.cuda.Event(True)
            v0.record(stream)  # replay() launches on the current stream
            vg.replay()
            v1.record(stream)
            torch.cuda.synchronize()
            vms = v0.elapsed_time(v1) / n
            del vg
            vb = w * h + out_w_v * out_h_v * out_bytes_px
            variants[name] = {"gpx_s": w * h / vms / 1e6, "us": vms * 1e3,
                              "hbm_gbs": vb / vms / 1e6, "frac": vb / vms / 1e6 / hbm_peak,
                              "alg_bytes": vb, "kernel_passes": passes}
            del vo

        for name, contract, pf in (("u8", "u8", 1), ("sr32", "sr32", 1),
                                   ("sr_prefetch_off", "sr", 0)):
            if contract == a.contract and pf == a.prefetch:
                continue
            variant(name, CONTRACT_PLANES[contract], ow, oh, OUT_BYTES[contract],
                    lambda d, vo, vp, sp, pf=pf: api.launch(d, pitch, w, h, taps, pf, vo, vp,
                                                        stream=sp))
        # detect path: replicate padding fused, same-size
        # u8 edge map; normalize = 2 stencil passes + threshold table
        variant("detect_pad_clamp_abs", ("u8",), w, h, 1,
                lambda d, vo, vp, sp: api.detect_device(d, pitch, w, h, taps, 1, True,
                                                    api.SaveMode.clamp_abs, vo, vp, scratch,
                                                    stream=sp))
        variant("detect_pad_normalize", ("u8",), w, h, 1,
                lambda d, vo, vp, sp: api.detect_device(d, pitch, w, h, taps, 1, True,
                                                    api.SaveMode.normalize, vo, vp, scratch,
                                                    stream=sp), passes=2)
        variant("sr_pad", CONTRACT_PLANES["sr"], w, h, OUT_BYTES["sr"],
                lambda d, vo, vp, sp: api.launch_ex(d, pitch, w, h, taps, 1, True, vo, vp,
                                                stream=sp))
        # non-default FilterParams: (1,1,1,1) fits the int16 lanes (packed
        # kernel, runtime taps), (2,3,5,7) the FP32 lanes (f32x2 kernel),
        # (1,32768,1,1) neither (generic 32-bit kernel)
        for prm in ((1, 1, 1, 1), (2, 3, 5, 7), (1, 32768, 1, 1)):
            tp = api.make_stream_taps(api.FilterParams(*prm))
            name = "sr_params_" + "_".join(map(str, prm))
            variant(name, CONTRACT_PLANES["sr"], ow, oh, OUT_BYTES["sr"],
                    lambda d, vo, vp, sp, tp=tp: api.launch(d, pitch, w, h, tp, 1, vo, vp,
                                                        stream=sp))
            variants[name]["kernel"] = api.kernel_for(tp)
        # 3x3 operator: Stream3Result gx+gy (int32) + g (f64)
        variant("sobel3_sr", ("gx", "gy", "g"), w - 2, h - 2, 16,
                lambda d, vo, vp, sp: api.launch3(d, pitch, w, h, 1, False, vo, vp, stream=sp))
        variant("sobel3_u8", ("u8",), w - 2, h - 2, 1,
                lambda d, vo, vp, sp: api.launch3(d, pitch, w, h, 1, False, vo, vp, stream=sp))
        if a.workload == "8k":
            # the u8 contracts are issue-bound: add the issue-rate roofline
            for name, key in (("u8", "8k/u8"), ("sobel3_u8", "8k/sobel3_u8")):
                if name in variants:
                    variants[name]["issue_roofline"] = issue_frac(key, variants[name]["us"])
        torch.cuda.empty_cache()

    # ---- smaller single images (C1 1080p, C2 4K), StreamResult contract ----
    # throughput: 50 launches in one CUDA graph over 4 rotating inputs (a
    # frame stream); latency: one launch then a host synchronize, wall clock
    # (the single-image case, launch overhead included), and the device time
    # of one launch alone (CUDA events), medians of 30
    sizes = {}
    if rank == 0 and frames == 1 and a.workload == "8k" and a.contract == "sr":
        for (sw, sh) in ((1920, 1080), (3840, 2160)):
            s_ins = []
            for i in range(4):
                d, sp_ = api.alloc_input(sw, sh, dev)
                api.synth_random_device(d, sp_, sw, sh, seed=77 + i, stream=s_ptr)
                s_ins.append(d)
            so, sop = api.alloc_planes(sw - 4, sh - 4, planes_names, dev)

            def one(i, st, sp_=sp_):
                api.launch(s_ins[i % 4], sp_, sw, sh, taps, a.prefetch, so, sop, stream=st)
            for i in range(5):
                one(i, s_ptr)
            torch.cuda.synchronize()
            n = 50
            vs = torch.cuda.Stream(dev)
            vs.wait_stream(stream)
            vg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(vg, stream=vs):
                for i in range(n):
                    one(i, vs.cuda_stream)
            vg.replay()
            torch.cuda.synchronize()
            v0, v1 = torch.cuda.Event(True), torch.cuda.Event(True)
            v0.record(stream)
            vg.replay()
            v1.record(stream)
            torch.cuda.synchronize()
            us_stream = v0.elapsed_time(v1) / n * 1e3
            del vg
            # single image: (a) the Python API call + synchronize, wall
            # clock; (b) the same launch as a one-node CUDA graph (what a
            # latency-bound C/C++ caller replays), replay + synchronize wall
            # clock and its device time (events around the replay)
            g1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1, stream=vs):
                one(0, vs.cuda_stream)
            g1.replay()
            torch.cuda.synchronize()
            wall_api, wall_graph, dev_us = [], [], []
            for i in range(30):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                one(i, s_ptr)
                torch.cuda.synchronize()
                wall_api.append((time.perf_counter() - t0) * 1e6)
                t0 = time.perf_counter()
                g1.replay()
                torch.cuda.synchronize()
                wall_graph.append((time.perf_counter() - t0) * 1e6)
                v0.record(stream)
                g1.replay()
                v1.record(stream)
                torch.cuda.synchronize()
                dev_us.append(v0.elapsed_time(v1) * 1e3)
            del g1
            # the same frames as ONE batched launch (sobel5_launch_batch, the
            # C4 path): 16 frames per launch, 4 launches in a graph
            nb = 16
            bi, bp = api.alloc_input(sw, sh, dev, frames=nb)
            for f_ in range(nb):
                api.synth_random_device(bi[f_], bp, sw, sh, seed=500 + f_, stream=s_ptr)
            bo, bop = api.alloc_planes(sw - 4, sh - 4, planes_names, dev, frames=nb)

            def batch(st, bi=bi, bp=bp, bo=bo, bop=bop):
                api.launch_batch(bi, bp, sh * bp, sw, sh, nb, taps, a.prefetch, bo, bop,
                                 (sh - 4) * bop, stream=st)
            batch(s_ptr)
            torch.cuda.synchronize()
            gb = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gb, stream=vs):
                for i in range(4):
                    batch(vs.cuda_stream)
            gb.replay()
            torch.cuda.synchronize()
            v0.record(stream)
            gb.replay()
            v1.record(stream)
            torch.cuda.synchronize()
            us_batch = v0.elapsed_time(v1) / (4 * nb) * 1e3
            del gb, bi, bo
            sb = sw * sh + (sw - 4) * (sh - 4) * OUT_BYTES[a.contract]
            sizes[f"{sw}x{sh}"] = {
                "stream_us_per_image": us_stream, "gpx_s": sw * sh / us_stream / 1e3,
                "frac": sb / us_stream / 1e3 / hbm_peak,
                "batch16_us_per_image": us_batch, "batch16_frac": sb / us_batch / 1e3 / hbm_peak,
                "latency_us_wall_api": float(np.median(wall_api)),
                "latency_us_wall_graph": float(np.median(wall_graph)),
                "latency_us_device": float(np.median(dev_us)), "alg_bytes": sb}
            del so, s_ins
        torch.cuda.empty_cache()

    # ---- e2e through the C ABI host entry with pinned buffers ----
    # Every rank runs it on its own image at the same time (each GPU has its
    # own PCIe link); the time is the max over ranks and the value the whole
    # job's pixels over it.
    e2e = None
    if not a.no_e2e and frames == 1 and a.workload != "32k-bands":
        import ctypes as C
        ctx = api.Context(local)
        h_in = torch.empty((h, w), dtype=torch.uint8, pin_memory=True)
        h_in.copy_(ins[0][:, :w].cpu())
        dt = {"gx": torch.int32, "gy": torch.int32, "gd": torch.int32, "gdt": torch.int32,
              "g": torch.float64, "g32": torch.float32, "u8": torch.uint8}
        h_out = {k: torch.empty((oh, ow), dtype=dt[k], pin_memory=True) for k in planes_names}
        pl = _abi.Planes(pitch=ow)
        for k, v in h_out.items():
            setattr(pl, k, v.data_ptr())
        diag = _abi.Diag()
        L = _abi.load()

        def e2e_call():
            st = L.sobel5_run_host(ctx.handle, h_in.data_ptr(), w, h, C.byref(taps), a.prefetch,
                                   C.byref(pl), C.byref(diag))
            api.check(st, "sobel5_run_host")

        for _ in range(3):
            e2e_call()
        n_e2e = max(5, min(a.steps, 30))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_call()
        t1 = time.perf_counter()
        el = t1 - t0
        if world > 1:
            t = torch.tensor([el], device="cpu" if a.share_gpu else dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        s_e2e = el / n_e2e
        # bytes that crossed PCIe device -> host in the last timed call, as
        # the library counts its copies (gx..gdt ride the int16 wire with the
        # default taps), and the bytes of the int32/f64 result planes
        d2h = int(L.sobel5_ctx_last_d2h_bytes(ctx.handle))
        result = sum(v.numel() * v.element_size() for v in h_out.values())
        narrow = ["gx", "gy", "gd", "gdt"] if d2h < result else []
        e2e = {"value": world * w * h / s_e2e / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": world * w * h, "d2h_bytes_per_step": world * d2h,
               "result_bytes_per_step": world * result,
               "ms_per_step": s_e2e * 1e3, "steps": n_e2e, "ranks": world,
               "path": "sobel5_run_host (C ABI), pinned host buffers, chunked H2D/kernel/D2H "
                       "overlap on 3 streams" +
                       (f"; {'/'.join(narrow)} cross PCIe as int16 and are sign-extended into "
                        "the int32 result planes by the host pool" +
                        (", which rebuilds g from them (exact; g does not cross PCIe)"
                         if d2h < result // 2 else "") if narrow else "") +
                       "; every rank one image, max time over ranks"}
        ctx.close()

    elif not a.no_e2e and frames > 1:
        # C4 end to end: the rank's frames from pinned host memory through
        # sobel5_run_host_frames (the frame-stream call: run_stream per frame,
        # pipelined across frames), 32 frames per call into one pinned
        # 32-frame output set; wall clock, max over ranks, whole-job frames
        import ctypes as C
        ctx = api.Context(local)
        h_in = torch.empty((frames, h, w), dtype=torch.uint8, pin_memory=True)
        d0 = ins[0]
        for f_ in range(frames):
            h_in[f_].copy_(d0[f_][:, :w].cpu())
        group = min(32, frames)
        dt = {"gx": torch.int32, "gy": torch.int32, "gd": torch.int32, "gdt": torch.int32,
              "g": torch.float64, "g32": torch.float32, "u8": torch.uint8}
        ho = {k: torch.empty((group, oh, ow), dtype=dt[k], pin_memory=True) for k in planes_names}
        pl = _abi.Planes(pitch=ow)
        for k, v in ho.items():
            setattr(pl, k, v.data_ptr())
        diag = _abi.Diag()
        L = _abi.load()

        def e2e_frames():
            d2h = 0
            for f0 in range(0, frames, group):
                n = min(group, frames - f0)
                st = L.sobel5_run_host_frames(ctx.handle, h_in[f0].data_ptr(), w, h, n, w * h,
                                              C.byref(taps), a.prefetch, C.byref(pl), ow * oh,
                                              C.byref(diag))
                api.check(st, "sobel5_run_host_frames")
                d2h += int(L.sobel5_ctx_last_d2h_bytes(ctx.handle))
            return d2h

        e2e_frames()
        n_e2e = 2
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            d2h = e2e_frames()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device="cpu" if a.share_gpu else dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        s_e2e = el / n_e2e
        result = sum(v[0].numel() * v.element_size() for v in ho.values()) * frames
        e2e = {"value": world * frames * w * h / s_e2e / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": world * frames * w * h,
               "d2h_bytes_per_step": world * d2h, "result_bytes_per_step": world * result,
               "ms_per_step": s_e2e * 1e3, "steps": n_e2e, "ranks": world,
               "path": f"sobel5_run_host_frames (C ABI) over the rank's {frames} frames, "
                       f"{group} frames per call, pinned input frames and output set, "
                       "int16 wire for gx..gdt; max time over ranks"}
        ctx.close()

    elif not a.no_e2e and a.workload == "32k-bands":
        # C5 end to end, every rank at once over its own PCIe link: its band's
        # input rows from pinned host memory, the band step (halo exchange
        # included), and every output plane's rows streamed back into pinned
        # host memory through a 256 MB staging buffer; wall clock, max over
        # ranks.
        h_body = torch.empty((plan.body_rows, pitch), dtype=torch.uint8, pin_memory=True)
        h_body.copy_(body.cpu())
        stage = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
        cur = torch.cuda.current_stream(dev)

        def e2e_step(i):
            with torch.cuda.stream(cur):
                body.copy_(h_body, non_blocking=True)
            step(i, s_ptr)
            with torch.cuda.stream(cur):
                d2h = 0
                for k, t in out.items():
                    flat = t[: plan.out_rows].reshape(-1).view(torch.uint8)
                    for o in range(0, flat.numel(), stage.numel()):
                        n = min(stage.numel(), flat.numel() - o)
                        stage[:n].copy_(flat[o:o + n], non_blocking=True)
                        d2h += n
            torch.cuda.synchronize()
            return d2h

        e2e_step(0)
        n_e2e = max(2, min(a.steps, 4))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(n_e2e):
            d2h = e2e_step(i + 1)
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device="cpu" if a.share_gpu else dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
            dd = torch.tensor([d2h], device="cpu" if a.share_gpu else dev, dtype=torch.float64)
            dist.all_reduce(dd)
            d2h = int(dd.item())
        s_e2e = el / n_e2e
        e2e = {"value": w * h / s_e2e / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": w * h, "d2h_bytes_per_step": d2h,
               "ms_per_step": s_e2e * 1e3, "steps": n_e2e, "ranks": world,
               "path": "RowBandPartition.run per rank: band rows H2D from pinned memory, band "
                       "kernel with halos, every output plane D2H through a 256 MB pinned "
                       "staging buffer; wall clock, max over ranks"}

    # the drop-in C++ API end to end (tools/cpp_e2e.cpp): sobel5::run_stream
    # returning freshly allocated StreamResult planes, as a reference user calls it
    e2e_cpp = None
    exe = os.path.join(ROOT, "build", "cpp_e2e")
    if rank == 0 and not a.no_e2e and frames == 1 and a.workload != "32k-bands" \
            and os.path.exists(exe):
        import subprocess
        try:
            r = subprocess.run([exe, str(w), str(h), "10"], capture_output=True, text=True,
                               timeout=300)
            d = json.loads(r.stdout.strip().splitlines()[-1])
            e2e_cpp = {"value": d["run_stream_gpx_s"], "unit": UNIT,
                       "ms_per_step": d["run_stream_ms"], "h2d_bytes_per_step": w * h,
                       "d2h_bytes_per_step": d["d2h_bytes"],
                       "path": "sobel5::run_stream (C++ drop-in, include/sobel5_b200), fresh "
                               "StreamResult planes per call",
                       "parts_ms": {k: d[k] for k in ("alloc_planes_ms", "run_host_pageable_ms",
                                                      "run_host_pinned_ms", "run_stream_3x3_ms")
                                    if k in d}}
        except Exception as ex:  # informative only
            e2e_cpp = {"error": str(ex)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:  # rank 0 at N=1 only
        cpu = cpu_reference(w, h, frames, a.cpu_seconds)
        cpu["host"] = host_cpu()
        if world == 1 and not a.no_cpu_matrix:
            cpu["matrix"] = cpu_matrix()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (synth_random generated on device, reference generator)",
            "config": base_config(a, world),
            "timing": {"timed_as": ("one CUDA graph of the K steps (captured after warm-up)"
                                    if use_graph else "Python launch loop"),
                       "l2": f"inputs rotated over {n_in} buffers ({n_in * in_bytes / 1e6:.0f} MB)"
                             f" + {rank_out_px * OUT_BYTES[a.contract] / 1e6:.0f} MB of "
                             "outputs per step and rank, both > 126 MB L2",
                       "hbm_gbs_achieved": achieved, **spread},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic,
                         "traffic_ratio": traffic_ratio,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"
                         if peak_kind == "measured" else "fallback (B200_PROFILING.md)",
                         "alg_bytes_per_launch": alg_bytes,
                         "kernel": ("sobel5_packed_default_kernel" if taps_default
                                    else "sobel5_stream_kernel")
                         + (" (TMA band rows, 6-row bands, write-back stores)" if a.contract == "sr" and a.prefetch
                            and a.workload != "4k" and not (a.workload == "32k-bands" and world > 1)
                            else ""),
                         "kernel_us": ms_step * 1e3},
            "gpu_launches": launches,
            **({"share_gpu": "testing mode: all ranks on cuda:0 over gloo"} if a.share_gpu else {}),
            "clocks": clocks.summary(),
            "variants": variants,
            "sizes": sizes or None,
            "e2e": e2e,
            "e2e_cpp_api": e2e_cpp,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

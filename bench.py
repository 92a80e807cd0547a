#!/usr/bin/env python
"""Benchmark of the cafx-b200 compute-actor backend (BASELINE.json).

Headline (one JSON line, rank 0): BASELINE config 3 -- one 16384x16384 fp32
Mandelbrot request (max_iter 1000, x in [-0.75,-0.73], y in [0.10,0.12],
pixel centres) served by ONE context over N devices, metric Giter/s (sum of
escape counts / time). A "step" is one pass of the hot path over the whole
image.

  value : device-resident: every device's share of the image (1M-pixel row
          bands dealt cyclically, the product's planner) into
          its HBM, CUDA events on each device's launching stream, L2 flushed
          between steps (not timed); a step's time is the max over devices.
  e2e   : the same request through the public C ABI (cafxg_mandelbrot) into
          one pinned host image: the context's multi-device planner splits it,
          every device copies its bands into disjoint ranges of the image.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

--gpus N opens one context over devices 0..N-1 and fails loudly when fewer
are visible. Under torchrun, rank 0 runs the whole N-device request (the
north star: one compute actor served by every GPU of the box); the other
ranks only join the barriers (gloo: the path has no data-path collective).

`--impl reference` times the reference's CPU path on the host cores: the
unmodified reference's mandelbrot_cell (bench.cpp:367, compiled into
oracle/_ref) over a row sample of cfg3's region, in fp64 (its only
precision), plus its run_mandelbrot(16000, 500) at paper scale.
"""
from __future__ import annotations

import argparse
import ctypes
import datetime
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_IMG = H_IMG = 16384
MAX_ITER = 1000
REGION = (-0.75, -0.73, 0.10, 0.12)
BAND_ROWS = 64          # 64 x 16384 = 1M-pixel bands, the planner's band size
# CAFXG_VIRTUAL_DEVICES=V (tests only): the N-device code path on ONE GPU --
# the context presents V devices on device 0 (its own streams each), torch
# tensors of "device k" live on cuda:0. Never a measurement: the line says so.
VIRTUAL = int(os.environ.get("CAFXG_VIRTUAL_DEVICES", "0") or 0)


def phys(k: int) -> int:
    """CUDA ordinal behind context device k."""
    return 0 if VIRTUAL > 1 else k


def ctx_mask(n: int) -> int:
    return 1 if VIRTUAL > 1 else (1 << n) - 1
METRIC = "Mandelbrot Giter/s (BASELINE cfg3: 16384^2 fp32 max_iter=1000 zoom)"
WORKLOAD = ("cfg3: one 16384x16384 fp32 Mandelbrot request, max_iter=1000, "
            "x[-0.75,-0.73] y[0.10,0.12], pixel centres")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="cafxg", choices=["cafxg", "reference"])
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the cfg1/cfg2/cfg4/cfg5 side measurements")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---- clocks during the timed region ------------------------------------------------

class ClockSampler:
    """nvidia-smi sampled every 100 ms on the given GPUs while a timed region
    runs; median SM clock under load, max clock, throttle reasons seen."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus, self.proc, self.path = list(gpus), None, None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(map(str, self.gpus)),
                 f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "gpus": self.gpus}


# ---- distributed helpers -------------------------------------------------------------

class Dist:
    """Control plane only (barriers): rank 0 serves the whole N-device request
    through one context, so the ranks exchange nothing but a barrier; a CPU
    (gloo) group suffices."""

    def __init__(self, backend="gloo"):
        self.rank, self.world, self.local = env_rank()
        self.on = self.world > 1
        if self.on:
            import torch.distributed as dist
            dist.init_process_group(backend, timeout=datetime.timedelta(hours=2))
            self.dist = dist

    def barrier(self):
        if self.on:
            self.dist.barrier()

    def close(self):
        if self.on:
            self.dist.destroy_process_group()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def fp_peak_probe():
    """Runs tools/fp_peak (built by __graft_entry__.build) on device 0: the
    FP32/FP64 pipe throughput measured on this box (lane-ops/s), the
    roofline denominator next to the derived one."""
    exe = os.path.join(ROOT, "paper_1505_07368_b200", "tools", "fp_peak")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout
    except Exception:
        return None
    res = {}
    for line in out.splitlines():
        try:
            j = json.loads(line)
        except ValueError:
            continue
        if j.get("kind") == "FADD2 packed":
            res["fp32_lane_tops"] = j["lane_Tops"]
        elif j.get("kind") == "DADD":
            res["fp64_lane_tops"] = j["lane_Tops"]
    return res or None


# ---- CPU baselines (test infrastructure: oracle / oracle/_ref) -----------------------

def cpu_region_rate(x0, x1, y0, y1, w, h, it, target_s):
    """The reference's own escape loop (mandelbrot_cell, bench.cpp:367, from
    oracle/_ref; fp64) over a row sample of a region at pixel centres, every
    host thread: (Giter/s, cores, kind, sample text). Falls back to the fp32
    oracle port without oracle/_ref."""
    from oracle import oracle
    threads = os.cpu_count() or 1
    R = oracle.ref()

    def run(stride):
        if R is not None:
            sec = ctypes.c_double()
            iters = R.ref_region_iters_mt(x0, x1, y0, y1, w, h, it, stride, threads,
                                          ctypes.byref(sec))
            return float(iters), sec.value
        t0 = time.perf_counter()
        out = oracle.tile(x0, x1, y0, y1, w, h, it, fp64=False, centre=True,
                          threads=threads, sample_stride=stride)
        return float(out[::stride].sum(dtype="uint64")), time.perf_counter() - t0

    probe = max(1, h // 16)
    iters, dt = run(probe)
    per_row = iters / max(1, (h + probe - 1) // probe)
    rows = max(16, min(h, int(target_s * (iters / dt) / max(per_row, 1.0))))
    stride = max(1, h // rows)
    iters, dt = run(stride)
    reps = 1
    if stride == 1 and dt < target_s / 4:
        # the whole image is far below the target: time repeated full runs
        reps = max(2, min(50, int(target_s / max(dt, 1e-4))))
        t = [run(1)[1] for _ in range(reps)]
        dt = statistics.mean(t)
    what = ("the unmodified reference's mandelbrot_cell (bench.cpp:367, oracle/_ref, compiled "
            "from its sources with its own flags) in fp64 -- its only precision" if R is not None
            else "oracle port (cafx_oracle.c, -O3 -ffp-contract=off) in fp32")
    return iters / dt / 1e9, threads, "reference" if R is not None else "port", (
        f"{what}; every {stride}th row ({(h + stride - 1) // stride} rows x {w} px, "
        f"{iters:.3g} iterations in {dt:.3f} s" + (f", mean of {reps} runs" if reps > 1 else "")
        + f"), {threads} threads; {cpu_model()}")


def reference_paper_scale():
    """The unmodified reference's run_mandelbrot(16000, 500) (bench.cpp:481),
    all host threads, when oracle/_ref was built."""
    from oracle import oracle
    R = oracle.ref()
    if R is None or os.environ.get("CAFXG_SKIP_PAPER_SCALE"):
        return None
    workers = os.cpu_count() or 1
    ms = ctypes.c_double()
    chk = R.ref_run_mandelbrot(16000, 500, workers, ctypes.byref(ms))
    return {"call": "run_mandelbrot(16000, 500)", "wall_clock_ms": round(ms.value, 1),
            "checksum": str(chk), "workers": workers,
            "published": "3.2 s on 64 Opteron cores (PAPER.md:897)"}


def cpu_sgemm(n, A, B, target_s):
    """Threaded blocked fp32 matmul (oracle/sgemm_oracle.c, the builder-written
    CPU baseline: the reference has no matmul code) over a sample of row
    blocks of C = A.B, every host thread; extrapolated to the whole product
    when sampled. Returns (TFLOP/s, cores, sample text, rows, full)."""
    import numpy as np

    from oracle import oracle
    L = oracle.lib()
    threads = os.cpu_count() or 1
    block = 16

    def run(rows):
        C = np.empty((rows, n), dtype=np.float32)
        t0 = time.perf_counter()
        L.oracle_sgemm_f32_mt(A.ctypes.data, B.ctypes.data, C.ctypes.data, n, n, n, n, n, 0,
                              rows, block, threads)
        return time.perf_counter() - t0

    rows = min(n, threads * block)
    dt = run(rows)
    per_row = dt / rows
    rows = max(rows, min(n, int(target_s / per_row) // (threads * block) * threads * block))
    reps = 1
    if rows >= n and n * per_row < target_s / 4:
        reps = max(2, min(50, int(target_s / (n * per_row))))
    dt = statistics.mean(run(rows) for _ in range(reps))
    tflops = 2.0 * rows * n * n / dt / 1e12
    full = rows >= n
    sample = (f"oracle_sgemm_f32_mt (threaded blocked fp32, auto-vectorised -O3), rows "
              f"[0, {rows}) of C = {rows} x {n} x {n} in {dt:.3f} s"
              + (f" (mean of {reps} runs)" if reps > 1 else "") + f", {threads} threads; "
              + ("the whole product" if full else
                 f"extrapolated: the full {n}^3 product would take "
                 f"{dt * n / rows:.1f} s") + f"; {cpu_model()}")
    return tflops, threads, sample, rows, full


# ---- the reference arm ------------------------------------------------------------------

def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import oracle
    threads = os.cpu_count() or 1
    x0, x1, y0, y1 = REGION
    R = oracle.ref()

    # the reference's own escape loop (mandelbrot_cell, bench.cpp:367, from
    # oracle/_ref) over cfg3's region in fp64 (it has no fp32 path); the
    # oracle port in fp32 only when the reference could not be compiled
    def run(stride):
        if R is not None:
            sec = ctypes.c_double()
            it = R.ref_region_iters_mt(x0, x1, y0, y1, W_IMG, H_IMG, MAX_ITER, stride, threads,
                                       ctypes.byref(sec))
            return float(it), sec.value
        t0 = time.perf_counter()
        out = oracle.tile(x0, x1, y0, y1, W_IMG, H_IMG, MAX_ITER, fp64=False, centre=True,
                          threads=threads, sample_stride=stride)
        return float(out[::stride].sum(dtype="uint64")), time.perf_counter() - t0

    # size the per-step sample to ~4 s of CPU work
    it, dt = run(1024)
    rate, per_row = it / dt, it / (H_IMG // 1024)
    stride = max(1, H_IMG // max(16, min(H_IMG, int(4.0 * rate / per_row))))
    times, iters = [], 0.0
    for k in range(args.warmup + args.steps):
        it, dt = run(stride)
        if k >= args.warmup:
            times.append(dt)
            iters = it
    step_s = statistics.mean(times)
    value = iters / step_s / 1e9
    kind = "reference" if R is not None else "port"
    sample = (f"every {stride}th row of cfg3 ({H_IMG // stride} rows x {W_IMG} px, "
              f"{iters:.3g} iterations per step)")
    note = ("the unmodified reference's mandelbrot_cell (bench.cpp:367, oracle/_ref) in fp64 "
            "-- the reference has no fp32 path and hard-codes [-1.5,0.5]x[-1,1] in "
            "mandelbrot_row (bench.cpp:384-386), so its escape loop is driven over cfg3's "
            "pixel centres directly" if R is not None else
            "oracle port in fp32 (oracle/_ref not built)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Giter/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(step_s * 1e3, 2), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if R is not None else "f32",
        "data": "synthetic (deterministic plane grid)",
        "config": {"workload": WORKLOAD, "sample": sample},
        "cpu_baseline": {"value": round(value, 4), "unit": "Giter/s", "cores": threads,
                         "kind": kind, "sample": sample + "; " + note + "; " + cpu_model()},
        "e2e": {"value": round(value, 4), "unit": "Giter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    paper = reference_paper_scale()
    if paper:
        line["reference_paper_scale"] = paper
    print(json.dumps(line), flush=True)


# ---- our arm: the headline ------------------------------------------------------------------

def cfg3_device(ctx, ndev, fp64, steps, warmup, clocks=None):
    """Device-resident cfg3 over `ndev` devices: returns a dict with the step
    time (max over devices, mean over steps), per-device kernel times, the
    iterations, launches and a row spot check against the oracle."""
    import numpy as np
    import torch

    import paper_1505_07368_b200 as pkg
    from oracle import oracle
    from paper_1505_07368_b200.shard import band_tiles
    full = pkg.mandel_desc(*REGION, W_IMG, H_IMG, MAX_ITER, fp64=fp64, centre=True)
    tiles = [band_tiles(full, ndev, k, BAND_ROWS, global_offsets=False) for k in range(ndev)]
    npx = [sum(t.nrows * t.ncols for t in tk) for tk in tiles]
    outs = [torch.empty(npx[k], dtype=torch.int32, device=f"cuda:{phys(k)}") for k in range(ndev)]
    # 256 MiB per device written between steps (untimed): > the 126 MB L2
    flush = [torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{phys(k)}") for k in range(ndev)]
    # real streams: torch's default stream is the legacy NULL stream (handle
    # 0), which the C ABI would read as "use the context's own stream"
    streams = [torch.cuda.Stream(device=phys(k)) for k in range(ndev)]

    def launch_all():
        for k in range(ndev):
            ctx.mandelbrot_device(tiles[k], outs[k].data_ptr(), streams[k].cuda_stream, device=k)

    for _ in range(max(warmup, 1)):
        launch_all()
    for k in range(ndev):
        torch.cuda.synchronize(phys(k))
    iters_dev = [float(o.to(torch.int64).sum().item()) for o in outs]
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(ndev)] for _ in range(steps)]
    for k in range(ndev):
        torch.cuda.synchronize(phys(k))
    st0 = ctx.stats()
    if clocks:
        clocks.start()
    for s in range(steps):
        for k in range(ndev):
            with torch.cuda.stream(streams[k]):
                flush[k].zero_()                  # L2 flush, before the start event
                ev[s][k][0].record(streams[k])
        launch_all()
        for k in range(ndev):
            ev[s][k][1].record(streams[k])
    for k in range(ndev):
        torch.cuda.synchronize(phys(k))
    clk = clocks.stop() if clocks else None
    st1 = ctx.stats()
    per_dev = [[ev[s][k][0].elapsed_time(ev[s][k][1]) for s in range(steps)]
               for k in range(ndev)]
    step_ms = statistics.mean(max(per_dev[k][s] for k in range(ndev)) for s in range(steps))
    # spot check: three rows of the image, each from the device that owns it
    spot_ok = True
    rows_checked = []
    for r in (0, 4097, H_IMG - 1):
        band = r // BAND_ROWS
        k = band % ndev
        # position of the row inside device k's packed output
        local_band = band // ndev
        off = (local_band * BAND_ROWS + (r % BAND_ROWS)) * W_IMG
        got = outs[k][off:off + W_IMG].cpu().numpy().view(np.uint32)
        ref = oracle.tile(*REGION, W_IMG, H_IMG, MAX_ITER, fp64=fp64, centre=True, row0=r,
                          nrows=1)
        spot_ok = spot_ok and bool(np.array_equal(got, ref[0]))
        rows_checked.append(r)
    res = {"step_ms": step_ms, "iters": sum(iters_dev), "iters_dev": iters_dev,
           "kernel_ms_dev": [statistics.mean(v) for v in per_dev],
           "launches": int(st1.kernel_launches - st0.kernel_launches),
           "spot_ok": spot_ok, "rows_checked": rows_checked, "clocks": clk}
    del outs, flush
    torch.cuda.empty_cache()
    return res


def cfg3_e2e(ctx, fp64, steps, host):
    """cfg3 through the C ABI (cafxg_mandelbrot) into the pinned host image
    `host`: wall clock per request (median), bytes moved per request."""
    import paper_1505_07368_b200 as pkg
    full = pkg.mandel_desc(*REGION, W_IMG, H_IMG, MAX_ITER, fp64=fp64, centre=True)
    ctx.mandelbrot(full, host)  # warm-up
    st0 = ctx.stats()
    walls = []
    for _ in range(steps):
        t0 = time.perf_counter()
        ctx.mandelbrot(full, host)
        walls.append(time.perf_counter() - t0)
    st1 = ctx.stats()
    return {"ms": statistics.median(walls) * 1e3, "mean_ms": statistics.mean(walls) * 1e3,
            "h2d": (st1.h2d_bytes - st0.h2d_bytes) / steps,
            "d2h": (st1.d2h_bytes - st0.d2h_bytes) / steps,
            "devices_used": int(st1.devices_used)}


def run_ours(args):
    D = Dist()
    N = args.gpus
    if D.on and D.world != N:
        sys.exit(f"bench.py: --gpus {N} under a torchrun world of {D.world}")
    import torch
    visible = torch.cuda.device_count()
    if VIRTUAL > 1 and N == VIRTUAL and visible >= 1:
        visible = N  # test mode: N virtual devices on one GPU
    if N < 1 or N > visible:
        # fail loudly: a --gpus N run must not silently measure fewer devices
        sys.exit(f"bench.py: --gpus {N} but {visible} CUDA device(s) visible")
    if D.rank != 0:
        # rank 0's context serves the whole request on every device
        D.barrier()
        D.close()
        return
    line = measure(args, N, D)
    print(json.dumps(line), flush=True)
    D.barrier()
    D.close()


def measure(args, N, dist=None):
    import numpy as np
    import torch

    import paper_1505_07368_b200 as pkg
    from oracle import oracle
    probe = fp_peak_probe()
    ctx = pkg.Context(device_mask=ctx_mask(N))
    assert ctx.device_count == N, (ctx.device_count, N)
    torch.cuda.set_device(0)

    # ---- headline: cfg3 fp32, one request over N devices ----
    clocks = ClockSampler(sorted({phys(k) for k in range(N)}))
    dev = cfg3_device(ctx, N, False, args.steps, args.warmup, clocks)
    clk = dev["clocks"]
    step_ms = dev["step_ms"]
    iters = dev["iters"]
    value = iters / (step_ms / 1e3) / 1e9
    host = ctx.pinned_empty(W_IMG * H_IMG, np.uint32)
    e2e = cfg3_e2e(ctx, False, args.steps, host)
    e2e_value = iters / (e2e["ms"] / 1e3) / 1e9
    # the gathered image's spot rows against the oracle
    img = host.reshape(H_IMG, W_IMG)
    e2e_ok = all(np.array_equal(img[r], oracle.tile(*REGION, W_IMG, H_IMG, MAX_ITER,
                                                    fp64=False, centre=True, row0=r,
                                                    nrows=1)[0])
                 for r in (1, 8191, H_IMG - 2))
    # checksum of the gathered image: the compute-actor path's reply must
    # match it bit for bit (secondary "actor_requests_cafx")
    img_fnv = oracle.fnv1a_u32(host)

    # ---- roofline of the escape kernel (aggregate over the N devices) ----
    pk = peaks()
    sm_max = float(pk.get("sm_max_mhz") or 1965.0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    peak_gpu = sms * 128 * sm_max * 1e6 / 1e12
    achieved = 8.0 * iters / (step_ms / 1e3) / 1e12
    # DRAM traffic of the escape kernel from the committed ncu capture of the
    # full-image launch (profiles/round2/mandel_cfg3_mid_r2_full.txt:
    # 1.023902 GB written + 10.715136 MB read), the whole image over N devices
    traffic = round(1.023902e9 + 10.715136e6)
    # The same capture: FMA pipe busy 91.7% of active cycles over 33.71 ms at
    # 1.963 GHz = 6.31 executed lane-ops per iteration (6 in the unchecked
    # step, the rest block-end tests, refills and exact replays) against the
    # algorithmic 8.
    exec_ops_per_iter = 6.31
    roof = {"bound": "fp32_pipe", "achieved": round(achieved, 3),
            "peak": round(N * peak_gpu, 3), "unit": "TFLOP/s",
            "frac": round(achieved / (N * peak_gpu), 4), "traffic": traffic,
            "traffic_note": "dram read+write bytes per image (ncu, profiles/round2); "
                            "algorithmic output is 4 B/pixel",
            "ops_per_step": 8.0 * iters,
            "peak_basis": f"{N} x {sms} SMs x 128 FP32 lanes x {sm_max:.0f} MHz (sm_max_mhz of "
                          "MEASURED_PEAKS.json); algorithmic 8 FP ops per escape iteration "
                          "(3 mul + 5 add, SURVEY §8d)",
            "frac_executed": round(achieved / (N * peak_gpu) * exec_ops_per_iter / 8.0, 4),
            "frac_note": "frac counts the reference's 8 FP ops per iteration, so it can exceed "
                         "1: the kernel executes 6 per iteration (escape test deferred to the "
                         "ends of unchecked blocks, 2*zr*zi+ci as one FMA) plus block-end tests "
                         "and exact replays, 6.31 lane-ops/iteration measured (ncu FMA pipe "
                         "busy 91.7%, profiles/round2/mandel_cfg3_mid_r2_full.txt); "
                         "frac_executed is the pipe fraction doing that executed work"}
    if probe and probe.get("fp32_lane_tops"):
        pp = N * probe["fp32_lane_tops"]
        roof["peak_probe"] = round(pp, 3)
        roof["frac_probe"] = round(achieved / pp, 4)
        roof["frac_executed_probe"] = round(achieved / pp * exec_ops_per_iter / 8.0, 4)
        roof["probe_note"] = ("peak_probe = FADD2 lane-ops/s measured live on this box by "
                              "tools/fp_peak (full-occupancy packed adds) x N devices")
    if clk and clk.get("sm_mhz"):
        peak_clk = N * sms * 128 * clk["sm_mhz"] * 1e6 / 1e12
        roof["frac_at_measured_clock"] = round(achieved / peak_clk, 4)

    # ---- same precision as the reference: cfg3 in fp64 ----
    dev64 = cfg3_device(ctx, N, True, min(args.steps, 3), 1)
    v64 = dev64["iters"] / (dev64["step_ms"] / 1e3) / 1e9
    e2e64 = cfg3_e2e(ctx, True, 2, host)
    same = {"workload": "cfg3's region and size in fp64 (the reference's only precision), "
                        "bit-exact against the fp64 oracle (spot rows)",
            "value": round(v64, 3), "unit": "Giter/s", "ms_per_step": round(dev64["step_ms"], 3),
            "iterations_per_step": dev64["iters"],
            "e2e": {"value": round(dev64["iters"] / (e2e64["ms"] / 1e3) / 1e9, 3),
                    "ms_per_step": round(e2e64["ms"], 3)},
            "bit_exact_spot_check": dev64["spot_ok"],
            "roofline": {"bound": "fp64_pipe",
                         "achieved": round(8.0 * dev64["iters"] / (dev64["step_ms"] / 1e3)
                                           / 1e12, 3),
                         "peak": round(N * sms * 64 * sm_max * 1e6 / 1e12, 3),
                         "unit": "TFLOP/s"}}
    same["roofline"]["frac"] = round(same["roofline"]["achieved"] / same["roofline"]["peak"], 4)
    ctx.pinned_free(host)

    cpu = None
    if N == 1 and not args.no_cpu_baseline:
        v, cores, kind, desc = cpu_region_rate(*REGION, W_IMG, H_IMG, MAX_ITER, 12.0)
        cpu = {"value": round(v, 4), "unit": "Giter/s", "cores": cores, "kind": kind,
               "sample": desc}
        if kind == "reference":
            # both sides fp64: the same-precision speed-up
            same["cpu_baseline"] = dict(cpu)
            same["ratio_vs_cpu_reference"] = round(v64 / v, 1)
            same["e2e_ratio_vs_cpu_reference"] = round(same["e2e"]["value"] / v, 1)

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Giter/s", "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (deterministic plane grid, BASELINE cfg3)"
                + ("; VIRTUAL DEVICES on one GPU (code-path test, not a measurement)"
                   if VIRTUAL > 1 else ""),
        "config": {"workload": WORKLOAD,
                   "multi_device": f"one request, {N} device(s): one cafxg context over "
                                   f"devices 0..{N - 1}, 1M-pixel row bands dealt cyclically",
                   "iterations_per_step": iters,
                   "kernel_ms_per_device": [round(x, 3) for x in dev["kernel_ms_dev"]],
                   "l2": "256 MiB written per device between steps (untimed); "
                         "output 1 GiB > L2",
                   "bit_exact_spot_check": dev["spot_ok"] and e2e_ok},
        "e2e": {"value": round(e2e_value, 3), "unit": "Giter/s",
                "ms_per_step": round(e2e["ms"], 3), "h2d_bytes_per_step": int(e2e["h2d"]),
                "d2h_bytes_per_step": int(e2e["d2h"]),
                "devices_used_mask": e2e["devices_used"],
                "path": "cafxg_mandelbrot (C ABI) -> one pinned host image; the request is a "
                        "64-byte descriptor passed in kernel parameters, so h2d carries only "
                        "band tables; d2h is the 1 GiB image"},
        "gpu_launches": dev["launches"],
        "roofline": roof,
        "clocks": clk,
        "same_precision_fp64": same,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if not args.no_secondary:
        # the headline is complete here: a secondary that fails records its
        # error, and one that hangs (first N>1 run on real NVLink peers) cannot
        # take the headline with it -- the watchdog prints the line without the
        # unfinished secondaries, joins the ranks' barrier and exits
        dog = Watchdog(line, SECONDARY_BUDGET_S, dist)
        secondary = run_secondary(ctx, args, N, dog.out)
        guarded(secondary, "actor_requests_cafx",
                lambda: sec_actor_cafx(N, img_fnv, e2e["ms"]))
        dog.cancel()
        line["secondary"] = secondary
    try:
        ctx.close()
    except Exception as e:  # noqa: BLE001 -- e.g. a secondary left a sticky fault
        line.setdefault("secondary", {})["close_error"] = f"{type(e).__name__}: {e}"[:300]
    return line


# ---- our arm: the other configs -----------------------------------------------------------

def dev_time(fn, n, stream):
    import torch
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def median_wall(fn, n):
    fn()
    walls = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        walls.append(time.perf_counter() - t0)
    return statistics.median(walls) * 1e3


# seconds the secondaries may take after the headline is measured (a 1-GPU
# run needs ~60 s of them)
SECONDARY_BUDGET_S = float(os.environ.get("CAFXG_BENCH_SECONDARY_S", "900"))


class Watchdog:
    """Prints the headline line with the secondaries finished so far if they
    overrun their budget, then releases the other ranks and exits 0."""

    def __init__(self, line, budget_s, dist):
        import threading
        self.line, self.dist, self.out = line, dist, {}
        # the line is printed once: by the timer (which then exits) or, after
        # cancel(), by the caller
        self.lock, self.cancelled = threading.Lock(), False
        self.timer = threading.Timer(budget_s, self._fire)
        self.timer.daemon = True
        self.timer.start()

    def _fire(self):
        self.lock.acquire()   # held until os._exit: cancel() then never returns
        if self.cancelled:
            self.lock.release()
            return
        sec = dict(self.out)
        sec["watchdog"] = (f"secondaries stopped after {SECONDARY_BUDGET_S:.0f} s; "
                           "the entries present finished")
        self.line["secondary"] = sec
        print(json.dumps(self.line), flush=True)
        try:
            if self.dist is not None:
                self.dist.barrier()
        finally:
            os._exit(0)

    def cancel(self):
        self.timer.cancel()
        with self.lock:
            self.cancelled = True


def guarded(out, name, fn):
    """out[name] = fn(), or the error it raised: one failing secondary must not
    cost the others or the headline."""
    try:
        out[name] = fn()
    except Exception as e:  # noqa: BLE001 -- recorded in the line
        out[name] = {"error": f"{type(e).__name__}: {e}"[:500]}


def run_secondary(ctx, args, N, out=None):
    """cfg1/cfg2/paper scale (one-GPU configs) at N=1; cfg5 and cfg4 (the
    1/2/4/8-GPU configs) at every N on the N-device context; cfg3 through a
    compute actor."""
    out = {} if out is None else out
    if N == 1:
        guarded(out, "cfg1_mandelbrot_1920x1080_fp32", lambda: sec_cfg1(ctx, args))
        guarded(out, "cfg2_sgemm_1024", lambda: sec_sgemm(ctx, args, 1024, N))
        guarded(out, "paper_scale_run_mandelbrot_16000_500", lambda: sec_paper_scale(ctx))
    guarded(out, "cfg5_sgemm_16384", lambda: sec_sgemm(ctx, args, 16384, N))
    if N > 1:
        guarded(out, "cfg5_sgemm_16384_nccl_exchange", lambda: sec_sgemm_nccl(N))
    guarded(out, "cfg3_through_compute_actor", lambda: sec_cfg3_actor(ctx))
    try:
        out.update(sec_cfg4(ctx, args, N))
    except Exception as e:  # noqa: BLE001
        out["cfg4_request_storm"] = {"error": f"{type(e).__name__}: {e}"[:500]}
    return out


def sec_cfg1(ctx, args):
    import numpy as np
    import torch

    import paper_1505_07368_b200 as pkg
    stream = torch.cuda.Stream(device=0)
    d1 = pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100)
    o1 = torch.empty(1920 * 1080, dtype=torch.int32, device="cuda:0")
    ms = dev_time(lambda: ctx.mandelbrot_device(d1, o1.data_ptr(), stream.cuda_stream), 20,
                  stream)
    it1 = float(o1.to(torch.int64).sum().item())
    h1 = ctx.pinned_empty(1920 * 1080, np.uint32)
    e2e = median_wall(lambda: ctx.mandelbrot(d1, h1), 30)
    # the same request as one compute-actor request (cafxg_actor_enqueue) with
    # a pinned reply, the spawn_cl path
    actor = ctx.spawn("mandelbrot")
    descs = (pkg.MandelDesc * 1)(d1)
    act = median_wall(lambda: actor.request([descs], h1).result(timeout=60), 30)
    actor.release()
    ctx.pinned_free(h1)
    res = {"kernel_ms": round(ms, 4), "giter_s": round(it1 / ms / 1e6, 2),
           "e2e_ms": round(e2e, 4), "e2e_giter_s": round(it1 / e2e / 1e6, 2),
           "python_actor_e2e_ms": round(act, 4),
           "python_actor_path": "ComputeActor.request (ctypes, Future) -> cafxg_actor_enqueue, pinned reply; the C++ cafx path is secondary.actor_requests_cafx"}
    if not args.no_cpu_baseline:
        v, cores, kind, desc = cpu_region_rate(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100, 2.0)
        res["cpu_baseline"] = {"value": round(v, 4), "unit": "Giter/s", "cores": cores,
                               "kind": kind, "sample": desc}
        res["e2e_ratio_vs_cpu"] = round(res["e2e_giter_s"] / v, 1)
    return res


def sec_paper_scale(ctx):
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_mandelbrot.json")))
    want = [g for g in golden["run_mandelbrot"] if g["size"] == 16000][0]
    ctx.run_mandelbrot(16000, 500)
    runs = [ctx.run_mandelbrot(16000, 500) for _ in range(3)]
    return {
        "wall_clock_ms": round(min(r[1] for r in runs), 3),
        "checksum": str(runs[0][0]),
        "checksum_matches_reference": runs[0][0] == int(want["checksum"]),
        "path": "cafxg_run_mandelbrot: fp64 reference-mode image in HBM + device FNV-1a",
        "reference": "3.2 s on 64 Opteron cores (PAPER.md:897); "
                     f"{want['wall_clock_ms_8_workers_here'] / 1e3:.1f} s for the unmodified "
                     "reference on the 8-core build container"}


def sec_sgemm(ctx, args, n, N):
    """fp32 matmul C = A.B (cfg2: 1024^3, cfg5: 16384^3). Device-resident:
    each device's row block of A (M/N rows) times the whole of B, CUDA events
    per device, max over devices. End to end: cafxg_sgemm over the N-device
    context (1/N of B up per device; at N > 1 every device's GEMM reads the
    other slices from the peers in place -- peer_gemms -- or, without peer
    access, B is replicated by the NCCL all-gather)."""
    import numpy as np
    import torch

    from oracle import oracle
    A_h = oracle.fill_uniform(n * n, 1).reshape(n, n)
    B_h = oracle.fill_uniform(n * n, 2).reshape(n, n)
    rows = n // N
    streams = [torch.cuda.Stream(device=phys(k)) for k in range(N)]
    As = [torch.from_numpy(A_h[k * rows:(k + 1) * rows]).to(f"cuda:{phys(k)}") for k in range(N)]
    Bs = [torch.from_numpy(B_h).to(f"cuda:{phys(k)}") for k in range(N)]
    Cs = [torch.empty(rows, n, device=f"cuda:{phys(k)}") for k in range(N)]
    reps = 20 if n <= 2048 else 3

    def launch_all():
        for k in range(N):
            ctx.sgemm_device(rows, n, n, As[k].data_ptr(), Bs[k].data_ptr(), Cs[k].data_ptr(),
                             streams[k].cuda_stream, device=k)

    launch_all()
    for k in range(N):
        torch.cuda.synchronize(phys(k))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(N)]
    for k in range(N):
        ev[k][0].record(streams[k])
    for _ in range(reps):
        launch_all()
    for k in range(N):
        ev[k][1].record(streams[k])
    for k in range(N):
        torch.cuda.synchronize(phys(k))
    ms = max(ev[k][0].elapsed_time(ev[k][1]) for k in range(N)) / reps
    tflops = 2.0 * n ** 3 / (ms / 1e3) / 1e12
    samp = np.arange(0, n, max(1, n // 16), dtype=np.uint32)
    Cn = np.concatenate([c.cpu().numpy() for c in Cs])
    R = oracle.sgemm_ref_rows(A_h, B_h, samp, n, n)
    err = oracle.sgemm_rel_err(Cn, R, samp, n)
    del As, Bs, Cs
    torch.cuda.empty_cache()
    hA = ctx.pinned_empty((n, n), np.float32)
    hB = ctx.pinned_empty((n, n), np.float32)
    hC = ctx.pinned_empty((n, n), np.float32)
    hA[...] = A_h
    hB[...] = B_h
    st0 = ctx.stats()
    e2e = median_wall(lambda: ctx.sgemm(hA, hB, hC), 30 if n <= 2048 else 3)
    st1 = ctx.stats()
    err_e2e = oracle.sgemm_rel_err(hC, R, samp, n)
    bf16 = float(peaks().get("bf16_tflops") or 1590.0)
    bf16s = float(peaks().get("bf16_tflops_sustained") or bf16)
    peak3 = N * bf16 / 2 / 3   # tf32 runs at half the bf16 rate; 3 MMAs per product
    res = {"kernel_ms": round(ms, 3), "tflops": round(tflops, 2), "n_gpus": N,
           "path": "3xTF32 tcgen05 (split + GEMM launches)"
                   + (f"; {N} devices, A row blocks, B on every device" if N > 1 else ""),
           "roofline": {"bound": "tensor", "achieved": round(tflops, 2),
                        "peak": round(peak3, 1), "unit": "TFLOP/s",
                        "frac": round(tflops / peak3, 4),
                        "frac_vs_sustained": round(tflops / (N * bf16s / 6), 4),
                        "peak_basis": f"{N} x measured bf16 {bf16} TF/s / 2 (tf32) / 3 "
                                      f"(hi*hi + hi*lo + lo*hi); sustained bf16 {bf16s}"},
           "e2e_ms": round(e2e, 3),
           "e2e_tflops": round(2.0 * n ** 3 / (e2e / 1e3) / 1e12, 2),
           "nccl_collectives": int(st1.nccl_collectives - st0.nccl_collectives),
           # N > 1: GEMMs that read B's K slices from the peers in place (no all-gather)
           "peer_gemms": int(st1.peer_gemms - st0.peer_gemms),
           "max_rel_err_sampled_rows": err, "max_rel_err_e2e": err_e2e, "tolerance": 1e-5}
    if N == 1 and not args.no_cpu_baseline:
        tf, cores, sample, srows, full = cpu_sgemm(n, A_h, B_h, 10.0)
        res["cpu_baseline"] = {"value": round(tf, 4), "unit": "TFLOP/s", "cores": cores,
                               "kind": "port", "sample": sample,
                               "extrapolated": not full}
        res["e2e_ratio_vs_cpu"] = round(res["e2e_tflops"] / tf, 1)
    for h in (hA, hB, hC):
        ctx.pinned_free(h)
    return res


def sec_sgemm_nccl(N, n=16384):
    """N > 1: cfg5 end to end on a second N-device context opened with
    CAFXG_SGEMM_P2P=0, i.e. B replicated by the NCCL all-gather over NVLink
    (ncclCommInitAll over the N GPUs) before each device's GEMM -- the
    baseline the fused exchange (cfg5_sgemm_16384: every device's GEMM reads
    B's slices from the peers in place) is measured against."""
    import numpy as np

    import paper_1505_07368_b200 as pkg
    from oracle import oracle
    old = os.environ.get("CAFXG_SGEMM_P2P")
    os.environ["CAFXG_SGEMM_P2P"] = "0"   # read by cafxg_open, per context
    try:
        c2 = pkg.Context(device_mask=ctx_mask(N))
    finally:
        if old is None:
            os.environ.pop("CAFXG_SGEMM_P2P", None)
        else:
            os.environ["CAFXG_SGEMM_P2P"] = old
    try:
        A_h = oracle.fill_uniform(n * n, 1).reshape(n, n)
        B_h = oracle.fill_uniform(n * n, 2).reshape(n, n)
        hA = c2.pinned_empty((n, n), np.float32)
        hB = c2.pinned_empty((n, n), np.float32)
        hC = c2.pinned_empty((n, n), np.float32)
        hA[...] = A_h
        hB[...] = B_h
        st0 = c2.stats()
        e2e = median_wall(lambda: c2.sgemm(hA, hB, hC), 3)
        st1 = c2.stats()
        samp = np.arange(0, n, max(1, n // 16), dtype=np.uint32)
        R = oracle.sgemm_ref_rows(A_h, B_h, samp, n, n)
        res = {"e2e_ms": round(e2e, 3),
               "e2e_tflops": round(2.0 * n ** 3 / (e2e / 1e3) / 1e12, 2),
               "n_gpus": N,
               "nccl_collectives": int(st1.nccl_collectives - st0.nccl_collectives),
               "peer_gemms": int(st1.peer_gemms - st0.peer_gemms),
               "max_rel_err_e2e": oracle.sgemm_rel_err(hC, R, samp, n), "tolerance": 1e-5,
               "path": "cafxg_sgemm over an N-device context with CAFXG_SGEMM_P2P=0: 1/N of B "
                       "up per device, in-place ncclAllGather, then each device's GEMM"}
        for h in (hA, hB, hC):
            c2.pinned_free(h)
        return res
    finally:
        c2.close()


def sec_cfg3_actor(ctx):
    """cfg3 as ONE compute-actor request (cafxg_actor_enqueue, pinned reply):
    large requests leave the batching path for the multi-device wave planner."""
    import numpy as np

    import paper_1505_07368_b200 as pkg
    actor = ctx.spawn("mandelbrot")
    d = pkg.mandel_desc(*REGION, W_IMG, H_IMG, MAX_ITER)
    descs = (pkg.MandelDesc * 1)(d)
    out = ctx.pinned_empty(W_IMG * H_IMG, np.uint32)
    st0 = ctx.stats()
    ms = median_wall(lambda: actor.request([descs], out).result(timeout=300), 3)
    st1 = ctx.stats()
    actor.release()
    iters = float(out.sum(dtype=np.uint64))
    ctx.pinned_free(out)
    return {"e2e_ms": round(ms, 3), "giter_s": round(iters / ms / 1e6, 2),
            "devices_used_mask": int(st1.devices_used),
            "launches_per_request": (st1.kernel_launches - st0.kernel_launches) / 4,
            "path": "ComputeActor.request -> cafxg_actor_enqueue -> dispatcher -> row bands "
                    "over every device, overlapped waves"}


def sec_actor_cafx(N, cfg3_fnv, cfg3_e2e_ms):
    """cfg1 and cfg3 as single requests of a cafx scoped_actor (unmodified
    reference runtime) to a gpu_actor (tools/actor_request_cafx.cpp); replies
    checked against the oracle (cfg1) and the C-ABI image (cfg3) by FNV-1a."""
    import paper_1505_07368_b200 as pkg
    from oracle import oracle
    exe = os.path.join(ROOT, "build", "tests", "actor_request_cafx")
    if not os.path.exists(exe):
        return {"skipped": "build/tests/actor_request_cafx not built (needs /root/reference)"}
    r = subprocess.run([exe, str(ctx_mask(N))], capture_output=True, text=True, timeout=600)
    try:
        j = json.loads(r.stdout.strip().splitlines()[-1])
    except (ValueError, IndexError):
        return {"error": (r.stderr or r.stdout)[-500:], "status": r.returncode}
    ref1 = oracle.fnv1a_u32(oracle.tile(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100, fp64=False,
                                        centre=True))
    j["cfg1"]["bit_exact_vs_oracle"] = int(j["cfg1"]["fnv"]) == ref1
    j["cfg3"]["bit_exact_vs_c_abi_image"] = int(j["cfg3"]["fnv"]) == cfg3_fnv
    j["cfg3"]["c_abi_e2e_ms"] = round(cfg3_e2e_ms, 3)
    j["cfg3"]["overhead_vs_c_abi"] = round(j["cfg3"]["median_ms"] / cfg3_e2e_ms - 1, 4)
    j["status"] = r.returncode
    j["path"] = ("cafx scoped_actor::request (unmodified reference runtime) -> gpu_actor "
                 "(include/cafxg/gpu_actor.hpp) -> cafxg_actor_enqueue; reply vector in pinned "
                 "pool memory written by the device")
    del pkg
    return j


def storm_descs(total, seed=2024):
    """cfg4's request list: 64x64 fp64 tiles (pitch 1/512, max_iter 256) at
    seeded offsets inside [-2,1]x[-1,1]."""
    import numpy as np

    import paper_1505_07368_b200 as pkg
    rng = np.random.default_rng(seed)
    kx = rng.integers(0, 3 * 512 - 64 + 1, size=total)
    ky = rng.integers(0, 2 * 512 - 64 + 1, size=total)
    arr = np.zeros(total, dtype=np.dtype(pkg.MandelDesc))
    arr["x0"] = -2.0 + kx / 512
    arr["x1"] = arr["x0"] + 0.125
    arr["y0"] = -1.0 + ky / 512
    arr["y1"] = arr["y0"] + 0.125
    for f in ("width", "height", "nrows", "ncols"):
        arr[f] = 64
    arr["max_iter"] = 256
    arr["precision"] = 1
    arr["sampling"] = 1
    return arr


def sec_cfg4(ctx, args, N, clients=64, per=1600):
    """BASELINE config 4: 64 clients x 1600 64x64 fp64 tiles. The expected
    replies come from the unmodified reference's mandelbrot_cell over every
    tile (the CPU baseline, timed), and EVERY reply of every mode is checked
    against them."""
    import numpy as np

    import paper_1505_07368_b200 as pkg
    from oracle import oracle
    total = clients * per
    arr = storm_descs(total)
    descs = (pkg.MandelDesc * total).from_buffer(arr)
    ref = oracle.ref_tiles(descs, total)
    if ref is None:  # no oracle/_ref: the fp64 oracle port gives the expectation
        t0 = time.perf_counter()
        expect = np.concatenate([oracle.tile(d.x0, d.x1, d.y0, d.y1, 64, 64, 256, fp64=True,
                                             centre=True, threads=1).ravel() for d in descs])
        cpu_s, kind = time.perf_counter() - t0, "port"
    else:
        expect, _, cpu_s = ref
        kind = "reference"
    expect = expect.reshape(total, 4096)
    out = {}
    cores = os.cpu_count() or 1
    cpu = {"value": round(total / cpu_s, 1), "unit": "requests/s", "cores": cores, "kind": kind,
           "sample": f"all {total} tiles ({float(expect.sum(dtype=np.uint64)):.3g} iterations) "
                     f"through the reference's mandelbrot_cell in fp64 on {cores} threads in "
                     f"{cpu_s:.2f} s (tiles claimed one at a time); {cpu_model()}"}
    replies = ctx.pinned_empty((total, 4096), np.uint32)
    S = ctypes.CDLL(os.path.join(ROOT, "paper_1505_07368_b200", "libcafxg_storm.so"))
    S.cafxg_storm_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_uint32)]
    names = {0: "open loop (async sends), 64 native client threads",
             2: "closed loop (1 outstanding/client), clients as actors on %d worker threads"
                % cores,
             1: "closed loop (1 outstanding/client), one OS thread per client"}
    keys = {0: "cfg4_request_storm", 2: "cfg4_request_storm_closed_loop",
            1: "cfg4_request_storm_closed_loop_os_threads"}
    for mode in (0, 2, 1):
        actor = ctx.spawn("mandelbrot")
        wms, errs = ctypes.c_double(), ctypes.c_uint32()
        S.cafxg_storm_run(actor.handle, descs, replies.ctypes.data, 16384, clients, per,
                          mode, ctypes.byref(wms), ctypes.byref(errs))   # warm-up
        replies[:] = 0
        st0 = ctx.stats()
        rc = S.cafxg_storm_run(actor.handle, descs, replies.ctypes.data, 16384, clients, per,
                               mode, ctypes.byref(wms), ctypes.byref(errs))
        st1 = ctx.stats()
        actor.release()
        dt = wms.value / 1e3
        bad = int((replies != expect).any(axis=1).sum())
        out[keys[mode]] = {
            "mode": names[mode], "requests": total, "clients": clients, "n_gpus": N,
            "status": rc, "wall_ms": round(wms.value, 2),
            "requests_per_s": round(total / dt, 1),
            "giter_s": round(float(expect.sum(dtype=np.uint64)) / dt / 1e9, 2),
            "batches": int(st1.batches - st0.batches), "max_batch": int(st1.max_batch),
            "kernel_launches": int(st1.kernel_launches - st0.kernel_launches),
            "devices_used_mask": int(st1.devices_used),
            "errors": int(errs.value), "checked_tiles": total, "mismatched_tiles": bad}
        if mode == 0:
            out[keys[mode]]["cpu_baseline"] = cpu
            out[keys[mode]]["ratio_vs_cpu"] = round(total / dt / cpu["value"], 1)
    ctx.pinned_free(replies)
    # the drop-in itself: 64 cafx event-based client actors on the unmodified
    # reference runtime talking to one gpu_actor (tools/storm_cafx.cpp)
    exe = os.path.join(ROOT, "build", "tests", "storm_cafx")
    if os.path.exists(exe):
        with tempfile.TemporaryDirectory() as td:
            dpath, epath = os.path.join(td, "descs.bin"), os.path.join(td, "expect.u32")
            arr.tofile(dpath)
            expect.tofile(epath)
            # the reference scheduler with its default configuration, and with
            # CAFX_WORKERS set to the same worker count: left at 0, the
            # worker count is re-derived from std::thread::hardware_concurrency()
            # (a sysfs read) on every central enqueue and every steal sweep
            # (scheduler.hpp:39-44,143-145,353,385), which costs the closed loop
            # ~5x
            cores = str(os.cpu_count() or 1)
            base = {k: v for k, v in os.environ.items() if k != "CAFX_WORKERS"}
            for mode, workers in (("closed", None), ("closed", cores), ("open", None),
                                  ("open", cores)):
                cmd = [exe, dpath, epath, str(clients), str(per), mode, str(ctx_mask(N))]
                env = base if workers is None else dict(base, CAFX_WORKERS=workers)
                r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
                try:
                    j = json.loads(r.stdout.strip().splitlines()[-1])
                except (ValueError, IndexError):
                    j = {"error": (r.stderr or r.stdout)[-500:], "status": r.returncode}
                j["status"] = r.returncode
                j["n_gpus"] = N
                j["check"] = ("every reply memcmp'd with its tile's expected counts" if
                              mode == "closed" else
                              "every client's reply fingerprints == its expected tiles' "
                              "(multiset; async replies carry no request id)")
                j["path"] = ("cafx event_based_actor clients (unmodified reference runtime) "
                             "-> gpu_actor (include/cafxg/gpu_actor.hpp) -> libcafxg")
                j["cafx_workers_env"] = workers
                tag = "" if workers is None else "_cafx_workers_set"
                out[f"cfg4_request_storm_cafx_actors_{mode}_loop{tag}"] = j
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

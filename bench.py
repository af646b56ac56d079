"""Benchmark: coefficient-domain multi-Gabor matching pursuit on B200 (BASELINE.json metric).

One step = one full decomposition of the workload through the C ABI, i.e. the
paper's ``dgtrealmp_execute``: DGT analysis of every dictionary, the MP
loop until the stop rule, and the synthesis of the approximation.  The Gram
kernels are computed once per handle (``dgtrealmp_init``; excluded from
the paper's timings) and timed separately (``kernels_ms``).

Default workload: C2 = BASELINE.json configs[2], the metric's "5-dict multi-Gabor
L=220500 fp64" (run until 40 dB or 1e5 atoms).  value = MP iterations per second
of whole steps, summed over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--precision f64]
  python bench.py --impl reference ...   # the CPU oracle on the same workload
Multi-GPU (torchrun): independent replicas, one per GPU ("replicas only",
DESIGN.md §7); value = total iterations / max over ranks of the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import siggen  # noqa: E402

METRIC = "MP iterations/sec, 5-dict multi-Gabor L=220500 fp64; update GB/s vs HBM peak"
UNIT = "iterations/s"
HBM_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-steps", type=int, default=3)
    return ap.parse_args()


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return HBM_FALLBACK_GBS, "fallback"


def workload_desc(cfg, prec):
    ds = ",".join(f"{siggen.WINDOW_NAMES[d.win]}{d.gl}/a{d.a}/M{d.M}" for d in cfg.dicts)
    stop = f"K={cfg.maxit}" + (f", errdb={cfg.errdb}" if cfg.errdb != -math.inf else "")
    return f"{cfg.name}: L={cfg.Ls} {cfg.signal}(seed {cfg.seed}); dicts {ds}; thr={cfg.thr}; {stop}; {prec}"


# ---------------------------------------------------------------------------
# algorithmic bytes of the update: per selection, every entry of
# the subsampled kernel class box applied to every target dictionary reads and
# writes one coefficient and reads one kernel entry: 48 B (fp64) / 24 B (fp32).
# ---------------------------------------------------------------------------
def touched_per_atom(mp, dicts, atoms):
    W = len(dicts)
    total = np.zeros(atoms.size, dtype=np.int64)
    w, k, j = atoms["w"].astype(np.int64), atoms["m"].astype(np.int64), atoms["n"].astype(np.int64)
    for u in range(W):
        su = np.nonzero(w == u)[0]
        if su.size == 0:
            continue
        du = dicts[u]
        for v in range(W):
            dv = dicts[v]
            mu_lo, mu_hi, nu_lo, nu_hi = mp_boxes[(u, v)]
            nmu, nnu = mu_hi - mu_lo + 1, nu_hi - nu_lo + 1
            a_c, M_c = min(du.a, dv.a), max(du.M, dv.M)
            s_m, s_n = M_c // dv.M, max(1, dv.a // a_c)
            kp = k[su] * (M_c // du.M)
            on = (-(j[su] * (du.a // a_c)) - nu_lo) % s_n
            om = (-kp - mu_lo) % s_m
            nr = np.where(on < nnu, (nnu - on + s_n - 1) // s_n, 0)
            nc = np.where(om < nmu, (nmu - om + s_m - 1) // s_m, 0)
            total[su] += nr * nc
    return total


mp_boxes = {}


def loop_traffic(config, prec, kernel):
    """DRAM bytes (read + write) of one launch of the loop kernel from the committed ncu
    --set full capture (profiles/*loop_traffic.json), or None."""
    import glob
    key = f"{config}/{prec}/{kernel}"
    for fn in sorted(glob.glob(os.path.join(ROOT, "profiles", "*loop_traffic.json")), reverse=True):
        try:
            d = json.load(open(fn))
        except Exception:  # noqa: BLE001
            continue
        if key in d:
            e = d[key]
            return int(e["dram_read_bytes"] + e["dram_write_bytes"]), os.path.relpath(fn, ROOT) + ": " + e["source"]
    return None, None


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle (reference arm and cpu_baseline) -- the only place bench.py runs oracle/
# ---------------------------------------------------------------------------
def oracle_step(cfg, x):
    import oracle
    from oracle import gabor, loop
    t0 = time.perf_counter()
    lay = gabor.layout(cfg.dicts, cfg.Ls)
    grids = gabor.analysis_all(x, cfg.dicts, lay)
    t1 = time.perf_counter()
    S = oracle.Setup(tuple(cfg.dicts), cfg.thr, cfg.Ls, lay, grids, oracle_step.K, float(np.dot(x, x)), x)
    r = loop.mp_run(S, cfg.maxit, cfg.errdb, want_gaps=False)
    t2 = time.perf_counter()
    gabor.synthesize(r.atoms, cfg.dicts, lay.L, cfg.Ls)
    t3 = time.perf_counter()
    return r.n, t3 - t0, {"dgt_s": t1 - t0, "loop_s": t2 - t1, "synth_s": t3 - t2}


def oracle_prepare(cfg):
    from oracle import gabor
    t = time.perf_counter()
    oracle_step.K = gabor.kernels(cfg.dicts, cfg.thr)
    return time.perf_counter() - t


def cpu_info():
    """CPU model as lscpu / /proc/cpuinfo report it (family/model/stepping added, since
    virtualised hosts often hide the marketing name) and the host's logical CPUs."""
    name, fam, mod, step = "unknown", "?", "?", "?"
    try:
        for ln in open("/proc/cpuinfo"):
            k, _, v = ln.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name" and name == "unknown":
                name = v
            elif k == "cpu family" and fam == "?":
                fam = v
            elif k == "model" and mod == "?":
                mod = v
            elif k == "stepping" and step == "?":
                step = v
    except Exception:  # noqa: BLE001
        pass
    return f"{name} (family {fam} model {mod} stepping {step}), nproc {os.cpu_count()}"


def baseline_record(value, secs_loop, iters, sample):
    """cpu_baseline: the oracle as it stands, one thread (the method is sequential; the
    paper's code is single-threaded); loop-only rate reported beside it."""
    return {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
            "cpu": cpu_info(), "nproc": os.cpu_count(),
            "loop_only_it_per_s": iters / secs_loop if secs_loop > 0 else None}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    x = siggen.signal(cfg)
    kern_s = oracle_prepare(cfg)
    for _ in range(args.warmup):
        oracle_step(cfg, x)
    iters, secs, parts = 0, 0.0, []
    for _ in range(args.steps):
        n, s, p = oracle_step(cfg, x)
        iters += n
        secs += s
        parts.append(p)
    value = iters / secs
    sample = (f"{args.steps} full decompositions of {cfg.name} (DGT + {iters // args.steps} iterations "
              f"+ synthesis) on {cpu_info()}; kernel precompute {kern_s:.2f} s excluded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_desc(cfg, "f64"),
                       "step": "DGT + MP loop to the stop rule + synthesis (dgtrealmp_execute); kernels per handle",
                       "iterations_per_step": iters // max(args.steps, 1), "parallelism": "cpu-1thread"},
            "cpu_baseline": baseline_record(value, sum(p["loop_s"] for p in parts), iters, sample),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "phases_s": {k: float(np.mean([p[k] for p in parts])) for k in parts[0]}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# multi-rank aggregation (replicas)
# ---------------------------------------------------------------------------
def aggregate(times_ms, counts, world, device=None):
    """Whole-job numbers over `world` replicas: every timed region is the MAX over ranks
    (the slowest replica bounds the job), every count the SUM.  Returns (times, counts) as
    Python floats; world == 1 returns them unchanged.  Works with any process group
    backend (nccl on the GPU box, gloo in the CPU tests)."""
    if world <= 1:
        return [float(t) for t in times_ms], [float(c) for c in counts]
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in times_ms], dtype=torch.float64, device=device)
    c = torch.tensor([float(v) for v in counts], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return t.tolist(), c.tolist()


# ---------------------------------------------------------------------------
# native arm
# ---------------------------------------------------------------------------
def run_native(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2202_12380_b200.build import build_library
    build_library()
    import paper_2202_12380_b200.mpgabor as mpg

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream()
    x_host = siggen.signal(cfg)
    xd = torch.from_numpy(x_host).to(dev)

    tk0 = torch.cuda.Event(enable_timing=True)
    tk1 = torch.cuda.Event(enable_timing=True)
    tk0.record(stream)
    mp = mpg.MPGabor(cfg.dicts, cfg.thr, args.precision)
    tk1.record(stream)
    torch.cuda.synchronize()
    kernels_ms = tk0.elapsed_time(tk1)
    W = len(cfg.dicts)
    for u in range(W):
        for v in range(W):
            mp_boxes[(u, v)] = mp.kernel_box(u, v)[0]
    maxit = cfg.maxit
    bufs = mp.alloc(maxit, cfg.Ls)
    y = torch.empty(cfg.Ls, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def step():
        res, (atoms, energy, _) = mp.run(xd, maxit, cfg.errdb, bufs=bufs, fetch=False)
        mpg.mpgabor_synth(mp.h, atoms, res.n_atoms, y, cfg.Ls)
        return res

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    loop_ms, iters = [], 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = mp.launch_count()
    t_wall = time.perf_counter()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()                        # L2 flushed between timed steps (outside the events)
            ev[i][0].record(stream)
            res = step()
            ev[i][1].record(stream)
            loop_ms.append(mp.last_timing()[2])
            iters += res.n_atoms
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall_s = time.perf_counter() - t_wall
    launches = mp.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = float(sum(step_ms))
    (t_ms_max,), (total_iters,) = aggregate([t_ms], [iters], world, dev)

    # roofline of the dominant kernel (the persistent loop): algorithmic bytes / loop time
    out = mp.run(xd, maxit, cfg.errdb, bufs=bufs)
    dgt_ms, init_ms, one_loop_ms = mp.last_timing()
    touched = touched_per_atom(mp, cfg.dicts, out.atoms)
    bpc = 48 if args.precision == "f64" else 24
    alg_bytes = int(touched.sum()) * bpc
    loop_mean_ms = float(np.mean(loop_ms))
    peak, peak_kind = peaks()
    achieved = alg_bytes / (loop_mean_ms * 1e-3) / 1e9
    kernel = "mp_loop_kernel" if out.rounds == out.n + 1 else "mp_multi_kernel"
    traffic, traffic_src = loop_traffic(cfg.name, args.precision, kernel)

    # end to end through the host-buffer C-ABI call (pinned host memory)
    import torch as _t
    xh = _t.from_numpy(x_host).pin_memory()
    atoms_h = _t.empty(maxit * 32, dtype=_t.uint8).pin_memory()
    energy_h = _t.empty(maxit + 1, dtype=_t.float64).pin_memory()
    y_h = _t.empty(cfg.Ls, dtype=_t.float64).pin_memory()
    hh = mpg.mpgabor_create(cfg.dicts, mpg.MPG_F64 if args.precision == "f64" else mpg.MPG_F32)
    mpg.mpgabor_kernels(hh, cfg.thr)
    mpg.mpgabor_decompose_host(hh, xh, maxit, cfg.errdb, atoms_h, energy_h, y_h)   # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_iters, e2e_ms, d2h = 0, 0.0, 0
    for _ in range(max(1, args.steps)):
        e0.record(stream)
        r = mpg.mpgabor_decompose_host(hh, xh, maxit, cfg.errdb, atoms_h, energy_h, y_h)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        e2e_iters += r.n_atoms
        d2h = r.n_atoms * 32 + (r.n_atoms + 1) * 8 + cfg.Ls * 8
    mpg.mpgabor_destroy(hh)
    (e2e_ms,), (e2e_iters,) = aggregate([e2e_ms], [e2e_iters], world, dev)
    e2e_value = e2e_iters / (e2e_ms * 1e-3)

    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": total_iters / (t_ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.precision, "data": "synthetic",
        "config": {"workload": workload_desc(cfg, args.precision),
                   "step": "DGT + MP loop to the stop rule + synthesis (dgtrealmp_execute); kernels per handle",
                   "iterations_per_step": int(out.n), "stop": out.stop_name,
                   "l2": "flushed between timed steps (256 MiB write outside the step events)",
                   "parallelism": "replicas" if world > 1 else "single-gpu",
                   "launch": mp.launch_info(), "kernels_ms": kernels_ms,
                   "phase_ms": {"dgt": dgt_ms, "init": init_ms, "loop": one_loop_ms},
                   "wall_s": wall_s},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind, "kernel": kernel, "rounds_per_launch": int(out.rounds),
                     "alg_bytes_per_launch": alg_bytes,
                     "touched_per_iter": float(touched.mean()), "bytes_per_touched": bpc,
                     "us_per_iter": 1e3 * loop_mean_ms / max(1, out.n)},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": cfg.Ls * 8, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        kern_s = oracle_prepare(cfg)
        it_c, s_c, s_loop = 0, 0.0, 0.0
        for _ in range(args.cpu_sample_steps):
            n, s, ph = oracle_step(cfg, x_host)
            it_c += n
            s_c += s
            s_loop += ph["loop_s"]
        line["cpu_baseline"] = baseline_record(
            it_c / s_c, s_loop, it_c,
            f"{args.cpu_sample_steps} full decompositions of {cfg.name} ({it_c // args.cpu_sample_steps} "
            f"iterations each, DGT + loop + synthesis, numpy synthesis included); oracle kernels "
            f"{kern_s:.2f} s excluded")
    mp.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = siggen.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "native":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
    else:
        run_native(args, cfg, rank, world, local_rank)
    if world > 1 and args.impl == "native":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the field-mapping hot path (BASELINE.json metric).

Workload (default, `--config c2`): BASELINE.json configs[1] -- XGC-like graded
poloidal-plane disk, disk_graded(1, 577, 0.6) = 1,000,519 source vertices ->
DEGAS2-like uniform disk(1, 577) = 1,000,519 targets, MLS degree 2, C4
("Wendland") weights a=2, AdaptiveRadius(12, h_src, 1.5), 8-component field
f_c = sin((c+1)x) cos(y) + 2.  Synthetic inputs (synth.py restates the
reference generators bit for bit).

One step = the whole hot path over that batch, inputs resident in HBM:
  source binning (grid build) -> target ordering -> adaptive radius count
  -> CSR scan -> fused fill + C4 weights + QR fit (operator build)
  -> 8-component operator apply   [-> NCCL all-gather of the target field, N>1]
value = targets mapped per second (whole job).  `e2e` = the same through the
public one-shot API (fit_point_cloud(sources, field, targets, spec),
pointwise.py:434) with pinned host tensors: H2D of sources/targets/field and
D2H of the result inside the timed region (the field's H2D overlaps the
selection and operator build on a side stream).

N>1 (torchrun): weak scaling -- every rank maps its own 1,000,519 targets
(the target disk rotated by a rank-dependent angle) against the replicated
source cloud, then the full target field is all-gathered to every rank.

`--impl reference`: the reference's own CPU kernels (oracle/_ref = the
reference's _ext.pyx compiled here) on all host cores, on a bounded sample.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "target points mapped/sec (search+MLS build, apply GB/s) at 1/2/4/8 B200 vs CPU"
C2_H = 0.001956233500370731  # synth.disk_graded(1, 577, 0.6).mean_edge_length (pinned in tests)
C1_H = 0.011486339741053897  # synth.square(99).mean_edge_length


# ---------------------------------------------------------------- inputs
def workload(config, rank=0):
    from paper_2510_18838_b200 import pointwise as P
    from paper_2510_18838_b200 import synth

    if config == "c2":
        src = synth.disk_graded(1.0, 577, 0.6).coords
        tgt = synth.disk(1.0, 577).coords
        if rank:
            a = 0.1 * rank  # weak scaling: a distinct target set per rank
            c, s = math.cos(a), math.sin(a)
            tgt = np.ascontiguousarray(tgt @ np.array([[c, s], [-s, c]]))
        X = synth.sincos_field(src, 8)
        spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0),
                         P.AdaptiveRadius(12, C2_H, 1.5))
        desc = {"workload": "C2: disk_graded(1,577,0.6) 1,000,519 sources -> disk(1,577) "
                            "1,000,519 targets per GPU, MLS degree 2, C4 (Wendland) a=2, "
                            "AdaptiveRadius(12, h_src, 1.5), 8-component field",
                "sources": int(src.shape[0]), "targets_per_gpu": int(tgt.shape[0]),
                "components": 8, "degree": 2, "rbf": "c4", "selection": "adaptive(12,h,1.5)"}
    elif config == "lattice1m":
        # SURVEY.md §3/§6 scale-up of C1: linspace(0,1,1000)^2 lattice -> 1M
        # random targets, degree 2, C4, FixedRadius(2h), h = 1/999
        side = np.linspace(0.0, 1.0, 1000)
        xx, yy = np.meshgrid(side, side)
        src = np.ascontiguousarray(np.column_stack([xx.reshape(-1), yy.reshape(-1)]))
        # targets keep 2h off the boundary: a corner target sees only 4 lattice
        # points inside 2h, which the reference rejects (UnderdeterminedError)
        h = 1.0 / 999.0
        tgt = np.random.RandomState(rank).uniform(2 * h, 1 - 2 * h, (1000000, 2))
        X = synth.sincos_field(src, 8)
        spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.FixedRadius(2 * h))
        desc = {"workload": "1M lattice linspace(0,1,1000)^2 -> 1M random targets in "
                            "[2h,1-2h]^2, MLS degree 2, C4 a=2, FixedRadius(2h), 8-component field",
                "sources": int(src.shape[0]), "targets_per_gpu": int(tgt.shape[0]),
                "components": 8, "degree": 2, "rbf": "c4", "selection": "fixed(2h)"}
    elif config == "c1":
        src = synth.square(99).coords
        tgt = np.random.RandomState(rank).uniform(0, 1, (10000, 2))
        X = synth.sincos_field(src, 1)
        spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.FixedRadius(2 * C1_H))
        desc = {"workload": "C1: square(99) 10,000 sources -> 10,000 random targets, MLS "
                            "degree 2, C4 a=2, FixedRadius(2h), scalar",
                "sources": 10000, "targets_per_gpu": 10000, "components": 1, "degree": 2,
                "rbf": "c4", "selection": "fixed(2h)"}
    else:
        raise SystemExit(f"unknown config {config}")
    return src, tgt, X, spec, desc


# --------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.timed_from = 0
        self.err = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError as exc:
            self.proc = None
            self.err = str(exc)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first_sample(self, timeout=5.0):
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            if self.proc.poll() is not None:
                self.err = (self.proc.stderr.read() or "")[-300:]
                break
            time.sleep(0.02)

    def mark_timed(self):
        self.timed_from = len(self.lines)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # samples from the timed region (plus the last warm-up sample when the
        # timed region is shorter than the sampling period)
        lines = self.lines[max(0, self.timed_from - 1):]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(sm)}
        if not sm and self.err:
            out["error"] = self.err
        return out


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "fallback": True}


def ncu_traffic():
    """DRAM bytes per kernel from the committed ncu --set full capture
    (profiles/traffic_*.json, newest round), or {}."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "traffic_*.json")))
    if not paths:
        return {}
    with open(paths[-1]) as f:
        d = json.load(f)
    d["file"] = os.path.relpath(paths[-1], ROOT)
    return d


def fit_flops(counts, k):
    """F(m,k) = 2mk^2 - (2/3)k^3 + 6mk + k^2 + m per target."""
    m = counts.astype(np.float64)
    return float(np.sum(2 * m * k * k - (2.0 / 3.0) * k ** 3 + 6 * m * k + k * k + m))


# ------------------------------------------------------------ b200 arm
# kernels launched by one device step (our own, counted from the launch
# sequence in device.py / libfieldmap.so and checked against the ncu launch
# list, profiles/): bbox pair 1; grid build: cell keys, scan, scatter,
# in-cell placement 4; target order: keys, scan, scatter 3; select: stats init +
# select 2; ordered offsets: gather counts + scan 2; build: stats init + one
# per non-empty size bucket (+1 if some support overflows its slot); apply 1
def launches_per_step(sel):
    buckets = int(np.count_nonzero(sel.bucket_count)) if sel.bucket_count is not None else 1
    return 1 + 4 + 3 + 2 + 2 + 1 + buckets + (1 if sel.n_overflow else 0) + 1


def b200_step(src_d, tgt_d, X_d, spec, marks):
    import torch

    from paper_2510_18838_b200 import device as D
    from paper_2510_18838_b200 import pointwise as P
    from paper_2510_18838_b200.pointwise import _r_max_device

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((name, e))

    mark("start")
    bs, bt = D.device_bboxes([src_d, tgt_d])  # one sync for both boxes
    cloud = D.SourceCloud(src_d, bbox=bs)
    mark("grid")
    perm = cloud.target_order(tgt_d)
    mark("order")
    sel = spec.selection
    dsel = D.adaptive(sel.min_points, sel.r0, sel.growth, _r_max_device(cloud, tgt_d, bt)) \
        if hasattr(sel, "min_points") else D.fixed(sel.r_c)
    cnt = D.select(cloud, tgt_d, dsel, perm, 0)
    mark("select")
    op, stats = D.build_operator(cloud, tgt_d, cnt, P._rbf_pair(spec.rbf), spec.degree, spec.lam,
                                 spec.centering)
    mark("build")
    Y = op.apply(X_d)
    mark("apply")
    return Y, op, cnt, stats, cloud


def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2510_18838_b200 import device as D
    from paper_2510_18838_b200 import pointwise as P
    from paper_2510_18838_b200.distributed import map_gathered, upload_replicated  # noqa: F401

    torch.cuda.set_device(local_rank)
    src, tgt, X, spec, desc = workload(args.config, rank)
    nt_local = tgt.shape[0]
    src_d, tgt_d, X_d = D.to_device(src), D.to_device(tgt), D.to_device(X)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    pending = []

    def step(marks):
        if world > 1:
            # blocks of this rank's targets; each block's rows pushed to the
            # peers (copy engines, NVLink) behind the next block's build, and
            # the exchange of this step completing under the next step
            # (distributed.map_gathered pipelined); the timed region ends
            # after the last exchange has completed
            if gg is not None:  # the rank's compute as a CUDA graph, then the pushes
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                marks.append(("start", e))
                Y, done = gg.step()
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                marks.append(("graph+push", e))
            else:
                Y, done = map_gathered(src_d, tgt_d, X_d, spec, nblocks=args.blocks,
                                       marks=marks, pipelined=True)
            pending.append(done)
            while len(pending) > 1:
                pending.pop(0)
            return Y, None, None, torch.zeros(1, dtype=torch.int32), (None, Y)
        if gt is not None:
            # the whole step replayed as one CUDA graph (device.GraphedTransfer):
            # bboxes + geometry on the host (one D2H), every kernel of the path
            # in the graph -- the same kernels and work as b200_step
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append(("start", e))
            Y = gt.run()
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append(("graph", e))
            return Y, None, None, torch.zeros(1, dtype=torch.int32), (None, Y)
        Y, op, cnt, stats, cloud = b200_step(src_d, tgt_d, X_d, spec, marks)
        return Y, op, cnt, stats, (cloud, Y)

    def eager_phases(warm=3, runs=5):
        """Phase split of the eager step (`runs` passes after `warm`): the
        roofline's per-kernel times when the timed step is a graph replay or
        the pipelined N > 1 step."""
        ph, last = {}, None
        for i in range(warm + runs):
            flush.zero_()
            m1 = []
            last = b200_step(src_d, tgt_d, X_d, spec, m1)
            torch.cuda.synchronize()
            for (a, ea), (b, eb) in zip(m1[:-1], m1[1:]):
                if i >= warm:
                    ph[b] = ph.get(b, 0.0) + ea.elapsed_time(eb) / runs
        return ph, last

    gt = D.GraphedTransfer(src_d, tgt_d, X_d, spec) if (world == 1 and not args.no_graph) \
        else None
    gg = None
    if world > 1 and not args.no_graph:
        from paper_2510_18838_b200.distributed import GraphedGather

        gg = GraphedGather(src_d, tgt_d, X_d, spec)

    sampler = ClockSampler(local_rank)
    with sampler:
        sampler.wait_first_sample()
        if gt is not None:  # eager phase split first (before the graph is captured)
            ph1, eager = eager_phases()
        for _ in range(args.warmup):
            Y, op, cnt, stats, extra = step([])
        torch.cuda.synchronize()
        if int(stats[0].item()) != 0:
            raise SystemExit(f"{int(stats[0].item())} fits failed in the benchmark workload")
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        phase = {}
        step_ms = []
        sampler.mark_timed()
        if world > 1:
            for d in pending:
                d.wait()
            pending.clear()
            torch.cuda.synchronize()
            dist.barrier()
            torch.cuda.synchronize()
            # pipelined steps: one event pair around the whole loop (L2
            # flushes included -- conservative), ended after the last exchange
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                flush.zero_()
                marks = []
                Y, op, cnt, stats, extra = step(marks)
                for (a, ea), (b, eb) in zip(marks[:-1], marks[1:]):
                    phase.setdefault(b, []).append((ea, eb))
            for d in pending:
                d.wait()
            e1.record()
            torch.cuda.synchronize()
            phase = {b: sum(ea.elapsed_time(eb) for ea, eb in v) for b, v in phase.items()}
            step_ms = [e0.elapsed_time(e1)]
        for _ in range(args.steps if world == 1 else 0):
            flush.zero_()  # L2 flush between timed steps (outside the step events)
            marks = []
            Y, op, cnt, stats, extra = step(marks)
            torch.cuda.synchronize()
            for (a, ea), (b, eb) in zip(marks[:-1], marks[1:]):
                phase[b] = phase.get(b, 0.0) + ea.elapsed_time(eb)
            step_ms.append(marks[0][1].elapsed_time(marks[-1][1]))
    if world > 1:
        dist.barrier()
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = nt_local * world * args.steps / (total_ms * 1e-3)

    graph_check = None
    if gg is not None:
        graph_check = gg.check()
        if not all(c["valid"] for c in graph_check):
            raise SystemExit(f"graphed step not valid for this workload: {graph_check}")
    if gt is not None:
        graph_check = gt.check()
        if not graph_check["valid"]:
            raise SystemExit(f"graphed step not valid for this workload: {graph_check}")
        Y1, op, cnt, stats, _c = eager
        extra = (_c, Y1)
        if os.environ.get("FM_CELLS_PER_POINT"):
            # a different grid density changes the supports' discovery order,
            # i.e. the rounding of the fits: equal to ~1e-12, not bitwise
            rel = ((Y1 - gt.Y).abs() / Y1.abs().clamp_min(1e-300)).max().item()
            print(f"graph vs eager (cells_per_point differs): max rel {rel:.3e}",
                  file=sys.stderr)
            if not rel < 1e-9:
                raise SystemExit("graphed and eager steps disagree")
        elif not torch.equal(Y1, gt.Y):
            raise SystemExit("graphed and eager steps disagree")
        phase = {"graph (whole step)": phase.get("graph", 0.0)}
        phase.update({f"eager {k}": v * args.steps for k, v in ph1.items()})
        build_ms, apply_ms = ph1["build"], ph1["apply"]
    if world > 1:
        # roofline inputs from eager passes on this rank (after the timed
        # region; the pipelined step interleaves builds and exchanges)
        ph1, eager = eager_phases()
        Y1, op, cnt, stats, _c = eager
        build_ms, apply_ms = ph1["build"], ph1["apply"]
    elif gt is None:
        build_ms = phase["build"] / args.steps
        apply_ms = phase["apply"] / args.steps
    # roofline inputs (per launch, from this run's own CUDA events)
    counts = cnt.counts.cpu().numpy()
    k = P.n_monomials(spec.degree, 2)
    flops = fit_flops(counts, k)
    C = X.shape[1]
    apply_bytes = op.algorithmic_bytes(C)
    peaks = measured_peaks()
    traffic = ncu_traffic()
    fp64_peak = D.fp64_probe() if rank == 0 else None

    # e2e through the public API with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        src_h = torch.from_numpy(src).pin_memory()
        tgt_h = torch.from_numpy(tgt).pin_memory()
        X_h = torch.from_numpy(X).pin_memory()
        def e2e_step():
            if world > 1:
                # sharded public API: this rank's rows, then the NCCL all-gather
                # of the full target field, then D2H
                # of the full target field on every device; each rank's host
                # reads back its own rows (the field is complete across the
                # ranks' hosts -- copying all of it to every host would cost
                # N x the PCIe traffic for the same data)
                # the replicated sources and source field: 1/N of the rows
                # over each rank's PCIe link, the rest over NVLink
                td = tgt_h.to("cuda", non_blocking=True)
                sd = upload_replicated(src_h)
                Xd = upload_replicated(X_h)
                Yf = map_gathered(sd, td, Xd, spec, nblocks=args.blocks)
                r0 = rank * nt_local
                Yh = torch.empty((nt_local, Yf.shape[1]), dtype=Yf.dtype, pin_memory=True)
                Yh.copy_(Yf[r0:r0 + nt_local], non_blocking=True)
                torch.cuda.current_stream().synchronize()
                return Yh.numpy()
            # one-shot transfer of the 8-component field (pointwise.py:434):
            # host pinned buffers in, pinned host result out
            return P.fit_point_cloud(src_h, X_h, tgt_h, spec).numpy()

        Yh = None
        for _ in range(max(3, args.warmup)):
            Yh = e2e_step()  # held like in the timed loop (two pinned results alive)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_steps = []
        for _ in range(args.steps):
            ts = time.perf_counter()
            Yh = e2e_step()
            e2e_steps.append(1e3 * (time.perf_counter() - ts))
        if os.environ.get("FM_E2E_DEBUG"):
            print("e2e per-step ms:", " ".join(f"{x:.2f}" for x in e2e_steps), file=sys.stderr)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
        e2e = {"value": nt_local * world * args.steps / e2e_s, "unit": "targets/s",
               "h2d_bytes_per_step": int(tgt.nbytes + (src.nbytes + X.nbytes) // world),
               "d2h_bytes_per_step": int(nt_local * C * 8),
               "ms_per_step": 1e3 * e2e_s / args.steps}
        if world > 1:
            e2e["bytes_note"] = ("per rank: its own targets + 1/N of the replicated sources "
                                 "and source field over PCIe (the rest over NVLink, "
                                 "distributed.upload_replicated); D2H = its own target rows")

    if rank != 0:
        return None
    cpu = None if (args.no_cpu or world > 1) else cpu_baseline(args, src, tgt, X, spec)
    par = None
    if not args.no_parity and world == 1:
        par = parity_block(src, tgt, X, spec, extra[0], tgt_d, cnt, op, extra[1])
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "targets/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": DATA,
        "config": bench_config(desc, world),
        "parallelism": f"target-sharded x{world}" + (
            " + NCCL all-gather of the target field" if world > 1 else ""),
        "phases_ms_per_step": {k2: v / args.steps for k2, v in phase.items()},
        # graphed step: bbox 1, binning 4, order 3, stats init + fused
        # select/buckets 2, offsets scan 1, build stats init 1, buckets, apply 1
        "gpu_launches": (launches_per_step(cnt) if gt is None else
                         13 + bin(gt.mask).count("1")) * args.steps,
        "graph": graph_check,
        "roofline": {
            "kernel": "k_build (C4 weights + Householder QR + operator row, supports from k_select)",
            "bound": "fp64",
            "achieved": flops / (build_ms * 1e-3) / 1e12,
            "peak": fp64_peak,
            "unit": "TFLOP/s",
            "frac": (flops / (build_ms * 1e-3) / 1e12) / fp64_peak if fp64_peak else None,
            "traffic": traffic.get("k_build_per_step"),
            "traffic_unit": f"DRAM bytes per step, ncu ({traffic.get('file')})",
            "note": "algorithmic FP64 flops F(m,k) summed over this step's supports; peak = "
                    "DFMA-chain probe measured in this run (MEASURED_PEAKS.json has no FP64 "
                    "figure); the build is issue/latency bound, not FP64 bound",
        },
        "roofline_apply": {
            "kernel": "k_apply (CSR SpMM, 8 components)",
            "bound": "hbm",
            "achieved": apply_bytes / (apply_ms * 1e-3) / 1e9,
            "peak": peaks.get("hbm_gbs"),
            "unit": "GB/s",
            "frac": apply_bytes / (apply_ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
            "traffic": traffic.get("k_apply_per_launch"),
            "traffic_unit": f"DRAM bytes per launch, ncu ({traffic.get('file')})",
            "algorithmic_bytes": apply_bytes,
            "note": "bytes = nnz*12 + nt*4 + ns*C*8 + nt*C*8 (SURVEY §8(d)); peak of measured"
                    if not peaks.get("fallback") else "peak of fallback",
        },
        "nnz": op.nnz,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": par,
        "clocks": sampler.summary(),
    }
    return line


# --------------------------------------------------- C3 / C4 / C5 configs
LARGE = ("c3", "c3mq", "c4", "c5")


def workload_large(config, rank, world, scale=1.0):
    """BASELINE.json configs[2..4].  `scale` shrinks
    the point counts (tests / quick checks); 1.0 is the configuration."""
    from paper_2510_18838_b200 import pointwise as P
    from paper_2510_18838_b200.distributed import shard_bounds

    if config in ("c3", "c3mq"):
        # 16M random sources -> 16M random targets, Gaussian / multiquadric,
        # AdaptiveRadius(12, 1.5/sqrt(N), 1.5), degree 2, scalar; the 16M
        # targets split across the ranks (strong scaling)
        n = int(16_000_000 * scale)
        src = np.random.RandomState(1).uniform(0, 1, (n, 2))
        lo, hi = shard_bounds(n, rank, world)
        tgt = np.ascontiguousarray(np.random.RandomState(2).uniform(0, 1, (n, 2))[lo:hi])
        X = np.sin(src[:, :1]) * np.cos(src[:, 1:]) + 2.0
        kind = P.RbfKind.GAUSSIAN if config == "c3" else P.RbfKind.MULTIQUADRIC
        spec = P.FitSpec(2, P.RadialBasisSpec(kind, a=2.0),
                         P.AdaptiveRadius(12, 1.5 / math.sqrt(n), 1.5))
        desc = {"workload": f"C3: {n} random sources -> {n} random targets (RandomState 1/2), "
                            f"{kind.name.lower()} a=2, AdaptiveRadius(12, 1.5/sqrt(N), 1.5), "
                            "degree 2, scalar, targets split across ranks",
                "sources": n, "targets_total": n, "components": 1, "degree": 2}
        return src, tgt, X, spec, desc, dict(scaling="strong", total=n, metric=None,
                                             applies=1, chunk=n, gather=False)
    if config == "c4":
        # 5-D distribution function: GNET-like tensor source grid 64^2 (space)
        # x 16^3 (velocity) on [0,1]^5 -> 64M random GTC-like targets, degree 1,
        # per-axis metric making the source lattice isotropic, operator built
        # once per step and applied to 32 successive fields
        ns_ax = [max(2, int(round(v * scale ** 0.2))) for v in (64, 64, 16, 16, 16)]
        axes = [np.linspace(0.0, 1.0, k) for k in ns_ax]
        g = np.meshgrid(*axes, indexing="ij")
        src = np.ascontiguousarray(np.stack([a.reshape(-1) for a in g], axis=1))
        n = int(64_000_000 * scale)
        lo, hi = shard_bounds(n, rank, world)
        rs = np.random.RandomState(4)
        tgt = np.ascontiguousarray(rs.uniform(0, 1, (n, 5))[lo:hi]) if scale < 1 else None
        if tgt is None:  # 64M x 5 at full scale: only this rank's rows
            tgt = np.empty((hi - lo, 5))
            done = 0
            while done < n:  # the same stream as uniform(0, 1, (n, 5)), row blocks
                k = min(4_000_000, n - done)
                blk = rs.uniform(0, 1, (k, 5))
                a, b = max(lo, done), min(hi, done + k)
                if a < b:
                    tgt[a - lo:b - lo] = blk[a - done:b - done]
                done += k
        v = src[:, 2:]
        X = (np.exp(-np.sum((v - 0.5) ** 2, axis=1) * 8.0) *
             (1.0 + 0.1 * np.sin(6.0 * src[:, 0]) * np.cos(6.0 * src[:, 1])))[:, None]
        hs = 1.0 / (ns_ax[0] - 1)
        metric = [1.0, 1.0] + [(ns_ax[2] - 1) * hs] * 3  # velocity spacing -> spatial spacing
        spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4, a=2.0),
                         P.AdaptiveRadius(12, hs, 1.5))
        desc = {"workload": f"C4: 5-D tensor source grid {'x'.join(map(str, ns_ax))} on [0,1]^5 "
                            f"-> {n} random targets (RandomState 4), per-axis metric "
                            f"{metric}, degree 1, C4 a=2, AdaptiveRadius(12, h, 1.5), operator "
                            "built once per step then applied to 32 fields",
                "sources": int(src.shape[0]), "targets_total": n, "components": 1,
                "degree": 1, "applies": 32}
        return src, tgt, X, spec, desc, dict(scaling="strong", total=n, metric=metric,
                                             applies=32, chunk=16_000_000, gather=False)
    if config == "c5":
        # 3-D degree 3, 128M targets per GPU (RandomState(5 + rank)) against a
        # replicated 16M random source cloud, all-gather of the full field
        ns = int(16_000_000 * scale)
        nt = int(128_000_000 * scale)
        src = np.random.RandomState(1).uniform(0, 1, (ns, 3))
        tgt = np.random.RandomState(5 + rank).uniform(0, 1, (nt, 3))
        X = (np.sin(3 * src[:, 0]) * np.cos(2 * src[:, 1]) * np.exp(src[:, 2]))[:, None] + 2.0
        h = ns ** (-1.0 / 3.0)
        spec = P.FitSpec(3, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.AdaptiveRadius(40, h, 1.5))
        desc = {"workload": f"C5: {ns} random 3-D sources (replicated) -> {nt} random targets "
                            "per GPU (RandomState 5+rank), degree 3 (k=20), C4 a=2, "
                            "AdaptiveRadius(40, N^-1/3, 1.5), scalar, all-gather of the full "
                            "target field",
                "sources": ns, "targets_per_gpu": nt, "components": 1, "degree": 3}
        return src, tgt, X, spec, desc, dict(scaling="weak", total=nt * world, metric=None,
                                             applies=1, chunk=16_000_000, gather=True)
    raise SystemExit(f"unknown config {config}")


def run_large(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2510_18838_b200 import device as D
    from paper_2510_18838_b200 import pointwise as P
    from paper_2510_18838_b200.distributed import gather_target_field

    torch.cuda.set_device(local_rank)
    src, tgt, X, spec, desc, meta = workload_large(args.config, rank, world, args.scale)
    if meta["metric"] is not None:  # the oracle sees the same IEEE products
        src = np.ascontiguousarray(src * np.asarray(meta["metric"]))
        tgt = np.ascontiguousarray(tgt * np.asarray(meta["metric"]))
    src_d, tgt_d, X_d = D.to_device(src), D.to_device(tgt), D.to_device(X)
    nt = tgt.shape[0]
    C = X.shape[1]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    Y = torch.empty((nt, C), dtype=torch.float64, device="cuda")
    rbf = P._rbf_pair(spec.rbf)
    sel = spec.selection
    need = 0 if hasattr(sel, "min_points") else P.n_monomials(spec.degree, src.shape[1])
    nnz = [0]

    def step(marks):
        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((name, e))

        mark("start")
        bs, bt = D.device_bboxes([src_d, tgt_d])
        cloud = D.SourceCloud(src_d, bbox=bs)
        dsel = D.adaptive(sel.min_points, sel.r0, sel.growth, P._r_max_device(cloud, tgt_d, bt)) \
            if hasattr(sel, "min_points") else D.fixed(sel.r_c)
        mark("grid")
        ops, checks = D.map_chunked(cloud, tgt_d, dsel, rbf, spec.degree, spec.lam,
                                    spec.centering, X_d, Y, meta["chunk"],
                                    keep=meta["applies"] > 1, min_required=need)
        nnz[0] = sum(o.nnz for _, _, o in ops) if ops else nnz[0]
        mark("map")
        for t in range(meta["applies"] - 1):  # the remaining timesteps' applies
            for c0, c1, op in ops:
                op.apply(X_d, out=Y[c0:c1])
        if meta["applies"] > 1:
            mark("applies")
        out = Y
        if meta["gather"] and world > 1:
            out = gather_target_field(Y, nt * world)
            mark("allgather")
        return out, checks, cloud

    sampler = ClockSampler(local_rank)
    with sampler:
        sampler.wait_first_sample()
        for _ in range(args.warmup):
            out, checks, cloud = step([])
        torch.cuda.synchronize()
        bad = [(c0, int(st[0].item())) for c0, sst, st in checks if int(st[0].item())]
        if any(sst[2] or sst[4] for _, sst, _ in checks) or bad:
            raise SystemExit(f"selection/fit failures in the benchmark workload: {bad}")
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler.mark_timed()
        phase, total = {}, 0.0
        for _ in range(args.steps):
            flush.zero_()
            marks = []
            out, checks, cloud = step(marks)
            torch.cuda.synchronize()
            for (a, ea), (b, eb) in zip(marks[:-1], marks[1:]):
                phase[b] = phase.get(b, 0.0) + ea.elapsed_time(eb)
            total += marks[0][1].elapsed_time(marks[-1][1])
    t = torch.tensor([total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total = float(t.item())
    value = meta["total"] * args.steps / (total * 1e-3)
    # sampled parity (outside the timed region): oracle on a uniform stride of
    # this rank's targets against the whole source set
    par = None
    if not args.no_parity and rank == 0:
        from oracle import parity

        from paper_2510_18838_b200.pointwise import _KIND_CODE

        stride = max(1, nt // args.parity_sample)
        idx = np.arange(0, nt, stride)
        ts = np.ascontiguousarray(tgt[idx])
        tsd = D.to_device(ts)
        cl = D.SourceCloud(src_d, bbox=D.device_bboxes([src_d])[0])
        dsel = D.adaptive(sel.min_points, sel.r0, sel.growth, P._r_max_device(cl, tgt_d)) \
            if hasattr(sel, "min_points") else D.fixed(sel.r_c)
        sl = D.select(cl, tsd, dsel, cl.target_order(tsd), need)
        off, sid, dist_, _w = D.support_csr(cl, tsd, sl)
        dev = {"off": off.cpu().numpy(), "idx": sid.cpu().numpy(), "dist": dist_.cpu().numpy(),
               "values": Y.cpu().numpy()[idx]}
        if sl.radii is not None:
            dev["radii"] = sl.radii.cpu().numpy()
            dev["status"] = sl.status.cpu().numpy()
        # r_max of the whole rank's target set (as the device run used)
        osel = ("adaptive", sel.min_points, sel.r0, sel.growth) if hasattr(sel, "min_points") \
            else ("fixed", sel.r_c)
        ref = parity.oracle_transfer(src, X, ts, spec.degree, _KIND_CODE[spec.rbf.kind],
                                     spec.rbf.a, osel, spec.lam, spec.centering,
                                     r_max=P._r_max(src, tgt) if hasattr(sel, "min_points")
                                     else None)
        par = parity.check_transfer(src, X, ts, spec.degree, _KIND_CODE[spec.rbf.kind],
                                    spec.rbf.a, osel, dev, spec.lam, spec.centering, ref=ref)
        par["sample"] = f"every {stride}-th of this rank's {nt} targets ({idx.size})"
    if rank != 0:
        return None
    return {
        "metric": METRIC, "value": value, "unit": "targets/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps,
        "higher_is_better": True, "scaling": meta["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded uniform clouds / tensor grid)",
        "config": bench_config(desc, world),
        "phases_ms_per_step": {k: v / args.steps for k, v in phase.items()},
        "nnz_per_rank": nnz[0] or None, "parity": par, "clocks": sampler.summary(),
        "e2e": None, "cpu_baseline": None,
    }


# ------------------------------------------------------- reference arm
_REF = {}  # state shared with forked workers (set before the fork, never pickled)


def _ref_chunk(bounds):
    """Worker: the reference's compiled kernels (oracle/_ref) on one chunk of
    the sampled targets -- PreparedTransfer's selection + weights
    (pointwise.py:233-296) and one fit_many per component (its apply
    re-solves per call, pointwise.py:418-431)."""
    b0, b1 = bounds
    st = _REF
    from oracle import ref

    E = ref.ext()
    g, spec, X, src = st["grid"], st["spec"], st["X"], st["src"]
    sel = spec.selection
    tg = st["tg"][b0:b1]
    if hasattr(sel, "min_points"):
        off, idx, dist, radii, status = E.adaptive_radius_supports(
            tg, g.points, float(g.lo[0]), float(g.lo[1]), g.dx, g.dy, g.nx, g.ny,
            g.cell_offsets, g.cell_items, sel.min_points, sel.r0, sel.growth, st["r_max"])
        w = np.empty(idx.shape[0])
        for i in range(tg.shape[0]):  # pointwise.py:266-269 (per-target weight loop)
            w[off[i]:off[i + 1]] = E.rbf_weights(st["kind"], spec.rbf.a, float(radii[i]),
                                                 dist[off[i]:off[i + 1]])
    else:
        off, idx, dist = E.fixed_radius_supports(
            tg, g.points, float(g.lo[0]), float(g.lo[1]), g.dx, g.dy, g.nx, g.ny,
            g.cell_offsets, g.cell_items, sel.r_c)
        w = E.rbf_weights(st["kind"], spec.rbf.a, sel.r_c, dist)  # pointwise.py:250
    w = np.abs(w)  # pointwise.py:301
    out = np.empty((tg.shape[0], X.shape[1]))
    for c in range(X.shape[1]):
        v, _c, _st = E.fit_many(tg, off, idx, w, src, st["Xc"][c], spec.degree, spec.lam,
                                spec.centering)
        out[:, c] = v
    return b0, out


class ReferenceCPU:
    """The reference CPU path on all host cores: one persistent fork pool
    (OPENBLAS_NUM_THREADS=1 per worker), targets in chunks.  Each step maps a
    uniform-stride sample of the WHOLE target set (every `stride`-th target,
    so the graded disk's cheap and expensive regions are both represented)
    and rebuilds the source PointGrid (locate.py:144-161, restated in
    oracle/pointgrid.py) -- the grid's time is charged at the sample's share
    of the full target set, because one grid serves all targets."""

    def __init__(self, src, tgt, X, spec, stride, procs=None):
        import multiprocessing as mp

        from oracle.oracle import r_max_for
        from oracle.pointgrid import OraclePointGrid
        from paper_2510_18838_b200.pointwise import _KIND_CODE

        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        self.procs = procs or (os.cpu_count() or 1)
        self.src, self.nt, self.stride = src, tgt.shape[0], max(1, int(stride))
        self.sample = np.ascontiguousarray(tgt[::self.stride])
        self.ns = self.sample.shape[0]
        _REF.update(grid=OraclePointGrid(src), r_max=r_max_for(src, tgt), spec=spec, X=X,
                    src=src, tg=self.sample, kind=_KIND_CODE[spec.rbf.kind],
                    Xc=[np.ascontiguousarray(X[:, c]) for c in range(X.shape[1])])
        nchunks = 8 * self.procs  # small chunks: load balance across the disk
        b = np.linspace(0, self.ns, nchunks + 1).astype(int)
        self.work = [(int(b0), int(b1)) for b0, b1 in zip(b[:-1], b[1:]) if b1 > b0]
        self.pool = mp.get_context("fork").Pool(self.procs) if self.procs > 1 else None

    def step(self):
        """Returns (seconds charged to the sample, values of the sample)."""
        from oracle.pointgrid import OraclePointGrid

        t0 = time.perf_counter()
        OraclePointGrid(self.src)  # the grid build of this transfer
        t_grid = time.perf_counter() - t0
        t1 = time.perf_counter()
        if self.pool is not None:
            parts = self.pool.map(_ref_chunk, self.work, chunksize=1)
        else:
            parts = [_ref_chunk(w) for w in self.work]
        t_map = time.perf_counter() - t1
        out = np.concatenate([p for _, p in sorted(parts, key=lambda x: x[0])])
        return t_grid * self.ns / self.nt + t_map, out

    def describe(self):
        return (f"every {self.stride}-th of the {self.nt} targets ({self.ns} targets, all "
                f"components) per step on {self.procs} forked processes (one persistent pool, "
                f"OPENBLAS_NUM_THREADS=1); source PointGrid rebuilt each step and charged at "
                f"{self.ns}/{self.nt} of its time; reference kernels = oracle/_ref (the "
                f"reference's _ext.pyx compiled with its own flags)")

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


def ref_stride(nt, procs):
    """Sample stride: about 25k targets per host process per step (a few
    seconds of CPU), never more than the whole set."""
    return max(1, int(math.ceil(nt / (25000.0 * max(1, procs)))))


def cpu_baseline(args, src, tgt, X, spec):
    from oracle import ref

    if not ref.available():
        return {"unavailable": "oracle/_ref not built"}
    procs = os.cpu_count() or 1
    rc = ReferenceCPU(src, tgt, X, spec, ref_stride(tgt.shape[0], procs), procs)
    try:
        dt, _ = rc.step()
    finally:
        rc.close()
    return {"value": rc.ns / dt, "unit": "targets/s", "cores": procs, "kind": "reference",
            "cpu_model": cpu_model(), "sample": rc.describe()}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    from oracle import ref

    src, tgt, X, spec, desc = workload(args.config, 0)
    if not ref.available():
        return {"impl": "reference", "unavailable": "oracle/_ref (the reference's compiled "
                "_ext.pyx) is not built"}
    procs = os.cpu_count() or 1
    rc = ReferenceCPU(src, tgt, X, spec, ref_stride(tgt.shape[0], procs), procs)
    try:
        for _ in range(args.warmup):
            rc.step()
        total = 0.0
        for _ in range(args.steps):
            dt, _ = rc.step()
            total += dt
    finally:
        rc.close()
    value = rc.ns * args.steps / total
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "targets/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": bench_config(desc, world),
        "cpu_baseline": {"value": value, "unit": "targets/s", "cores": procs,
                         "kind": "reference", "cpu_model": cpu_model(),
                         "sample": rc.describe()},
        "e2e": {"value": value, "unit": "targets/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


# ---------------------------------------------------------------- parity
def parity_block(src, tgt, X, spec, cloud, tgt_d, sel, op, Y):
    """The benchmarked workload checked against the CPU oracle (outside the
    timed region): neighbour CSR / radii / status bitwise, fit status equal,
    values <= 1e-10 relative (oracle/parity.py)."""
    from oracle import parity
    from paper_2510_18838_b200 import device as D
    from paper_2510_18838_b200.pointwise import _KIND_CODE

    off, idx, dist, _w = D.support_csr(cloud, tgt_d, sel)
    dev = {"off": off.cpu().numpy(), "idx": idx.cpu().numpy(), "dist": dist.cpu().numpy(),
           "values": Y.cpu().numpy(), "fit_status": op.status.cpu().numpy()}
    s = spec.selection
    if hasattr(s, "min_points"):
        dev["radii"] = sel.radii.cpu().numpy()
        dev["status"] = sel.status.cpu().numpy()
        osel = ("adaptive", s.min_points, s.r0, s.growth)
    else:
        osel = ("fixed", s.r_c)
    return parity.check_transfer(src, X, tgt, spec.degree, _KIND_CODE[spec.rbf.kind],
                                 spec.rbf.a, osel, dev, spec.lam, spec.centering)


DATA = "synthetic (reference mesh generators restated bitwise; fields sin((c+1)x)cos(y)+2)"


def bench_config(desc, world):
    """The `config` object -- identical for both arms."""
    return dict(desc, n_gpus=world, l2="flushed between timed steps (256 MiB write)")


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: run N ranks under
    torch.distributed.run on this node (127.0.0.1) and pass rank 0's line
    through."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=["c1", "c2", "lattice1m", "c3", "c3mq", "c4", "c5"],
                    default="c2")
    ap.add_argument("--scale", type=float, default=1.0,
                    help="c3/c4/c5: shrink the point counts by this factor (checks)")
    ap.add_argument("--parity-sample", type=int, default=20000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="N=1: launch the step eagerly instead of replaying its CUDA graph")
    ap.add_argument("--blocks", type=int, default=1,
                    help="N>1: target blocks per rank (all-gather pipelining depth)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist

            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        line = (run_large if args.config in LARGE else run_b200)(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

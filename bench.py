#!/usr/bin/env python
"""Benchmark of the element-local HDG hot path (BASELINE.json metric):

  HDG elements/s (build+condense+recover, fp64) at k=3

One step = K1 geometry + K2 node build + K3 condense + K5 recover (+ K6 u*
for C5) over the whole mesh, coefficient fields evaluated at the nodes inside
the step (as the reference evaluates its callbacks inside build). Default
workload: config C2 (k=3, 32^3 Kuhn box, 196,608 tets) on one GPU. With N
GPUs (torchrun) rank r owns z-slab r of a 32 x 32 x 32N box: per-GPU work is
fixed ("weak" scaling) and the element-local step has no data-path collective.

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the
engine stream; L2 (126 MB) is flushed by a 512 MB write between steps outside
the timed interval; per-kernel times come from events recorded around each
kernel on the same stream (hdg_b200_stage_times). Multi-GPU: barrier +
synchronize around the timed loop and the max over ranks.

`--impl reference` times the reference algorithm's CPU restatement
(oracle/, the reference itself cannot be compiled here: no Eigen3) on all
host cores over the same whole mesh, per step (see run_reference).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "HDG elements/s (build+condense+recover, fp64) at k=3; % of HBM/FP64 roofline"
FP64_PEAK_TFLOPS = 37.0   # measured DMMA peak on this pool's B200 (profiles/fp64_peaks_r01.jsonl)
FP64_PEAK_SOURCE = "profiles/fp64_peaks_r01.jsonl (mma.sync f64 microbenchmark; MEASURED_PEAKS.json has no FP64 entry)"


def ncu_traffic(kernel_prefix: str):
    """dram read+write bytes per launch of a kernel from the newest committed
    ncu launch list (profiles/r*_launches.csv), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_launches.csv")))
    if not files:
        return None, None
    vals = []
    for line in open(files[-1]):
        parts = line.strip().split(",")
        if len(parts) >= 5 and kernel_prefix in parts[1]:
            try:
                vals.append(float(parts[3]) + float(parts[4]))
            except ValueError:
                pass
    # the full-size launches (the e2e leg launches the same kernel on element chunks)
    return (max(vals) if vals else None), os.path.relpath(files[-1], ROOT)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# executed fp64 instructions per element of condense6_kernel<3> (ncu instruction
# counts of the committed capture profiles/r02f_ncu_k3v6_c2.txt)
K3_DMMA_PER_ELT = 466
K3_FP64_ALU_PER_ELT = 1564


def c_sms(dev) -> int:
    import torch
    return torch.cuda.get_device_properties(dev).multi_processor_count


# --------------------------------------------------------------- flop model
def k3_flops(k: int) -> float:
    """Algorithmic fp64 flops per element of the condense kernel as executed
    (unpadded counts, symmetric products counted once). The
    k >= 2 kernels (kernels_condense6.cuh, kernels_condense5.cuh) skip the rows of Chat_h that
    vanish structurally (modes of top degree: only the first n1 = dim P_{k-1}
    rows are nonzero), so Y_h, R'_h and the S update are counted on those rows
    only (the count of the algorithm actually executed, never a
    larger one); its skipping of zero blocks inside those rows is not counted."""
    n = (k + 1) * (k + 2) * (k + 3) // 6
    m = 2 * (k + 1) * (k + 2)
    n1 = k * (k + 1) * (k + 2) // 6 if k >= 2 else n   # nonzero rows of Chat_h (k <= 1: the dense kernel)
    f = 0.0
    f += 2 * 2.0 * n ** 3                 # two Gauss-Jordan inverses (M, S)
    f += 2.0 * n * n * m                  # Zp = Mi W^T
    f += 3 * 2.0 * n1 * n * n + 3 * 3 * 2.0 * n1 * n   # Y_# = Chat_# Mi, R'_# = g Y
    f += 3 * 2.0 * n * n1 * (n1 + 1) / 2  # S += sum_# R'_# Chat_#^T (lower, n1 x n1)
    f += 2.0 * n1 * n * m + 4 * 3 * 2.0 * n1 * n + (n - n1) * m   # V: W_l Z_l^T on the dense rows, T W on the rest
    f += 2.0 * n * n * m + 2.0 * n * n    # Vs = Si V, fs
    f += 2 * 2.0 * n * m * (m + 1) / 2    # W Zp and V^T Vs (lower)
    f += 2.0 * m * n                      # Cf
    return f


def k2_flops(k: int, nq: int) -> float:
    d3 = (k + 1) * (k + 2) * (k + 3) // 6
    nsym = d3 * (d3 + 1) // 2
    return 2.0 * nsym * nq * 2 + 2.0 * nsym * 4 + 2.0 * d3 * nq


def step_algorithmic_bytes(k: int, nq: int, sampled: bool) -> float:
    """B = 2 x 164 (elements, coords, facebyele, perm for build and
    for recover) + 3 nq 8 (kappa^-1, c, f samples; SAMPLED fields only)
    + (m^2 + m) 8 (C, Cf written) + m 8 (lambda gathered) + 4 d3 8 (q, u written)."""
    d3 = (k + 1) * (k + 2) * (k + 3) // 6
    m = 2 * (k + 1) * (k + 2)
    return 2 * 164 + (3 * nq * 8 if sampled else 0) + (m * m + m) * 8 + m * 8 + 4 * d3 * 8


STEP_KERNELS = ("face_area_kernel", "geometry_kernel", "reset_build_status", "tau_check", "quad_build",
                "condense", "rescue_kernel", "recover")


def ncu_step_traffic():
    """DRAM bytes of one full-size step (sum over the step's kernels, each the
    largest launch of its name) from the newest committed ncu launch list."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_launches.csv")))
    if not files:
        return None, None
    best = {}
    for line in open(files[-1]):
        parts = line.strip().split(",")
        if len(parts) < 5:
            continue
        try:
            b = float(parts[3]) + float(parts[4])
        except ValueError:
            continue
        for kn in STEP_KERNELS:
            if kn in parts[1]:
                best[kn] = max(best.get(kn, 0.0), b)
    return (sum(best.values()) if best else None), os.path.relpath(files[-1], ROOT)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and "Active" in r[4 + i]
                          and "Not" not in r[4 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------- reference arm
# The reference (C++/Eigen) cannot be built in this image, so its CPU path is
# timed through the oracle's restatement (oracle/, the one other place this file
# may execute it): the same config mesh built by the oracle alone
# (oracle.meshes; no product library is loaded in this process), compiled
# callbacks for C2/C5's fields, every stage of the reference path
# (build_element_matrices -> local_blocks -> condense -> local_recover) over
# contiguous element chunks on all host cores. In the reference-arm process
# the oracle is compiled -O3 -march=native for the host it runs on.
def oracle_workload(cfg, nz_layers=None):
    """(ExpandedMesh, tables, fields, tau, per-element lambda) of a config's
    mesh (the first nz_layers cell layers if given), oracle only."""
    from oracle import core
    from oracle.meshes import config_mesh
    coords, elements, dirichlet, neumann = config_mesh(cfg.n, cfg.problem.bc, cfg.perturb, cfg.seed)
    if nz_layers is not None and nz_layers < cfg.n:
        ne = 6 * cfg.n * cfg.n * nz_layers
        el = elements[:ne]
        verts, inv = np.unique(el, return_inverse=True)
        el_local = inv.reshape(el.shape).astype(np.int32)
        lf = [(0, 1, 2), (0, 1, 3), (0, 2, 3), (3, 1, 2)]
        tris = {}
        for K in range(ne):
            for l in range(4):
                t = tuple(el_local[K, list(lf[l])])
                tris.setdefault(tuple(sorted(t)), []).append(t)
        bdry = np.array([v[0] for v in tris.values() if len(v) == 1], dtype=np.int32)
        em = core.expand(np.asfortranarray(coords[verts]), np.asfortranarray(el_local), np.asfortranarray(bdry),
                         np.zeros((0, 3), np.int32))
    else:
        em = core.expand(coords, elements, dirichlet, neumann)
    k = cfg.k
    qd = 2 * k + 2
    t = core.tables(k, qd, qd)
    if cfg.problem.kappa == CONFIGS_C2_KAPPA():
        fields = core.c2_native_fields()
    else:
        from paper_1305_1489_b200.fields import compile_field
        fld = lambda e: core.Field.program(compile_field(e).ops, compile_field(e).consts)
        fields = (fld(cfg.problem.kappa), fld(cfg.problem.c), fld(cfg.problem.f))
    tau = core.Stabilization(np.full((em.n_elements, 4), float(cfg.tau)))
    d2 = (k + 1) * (k + 2) // 2
    # lambda: the GPU arm's smooth skeleton vector, gathered per element (gather_traces)
    uh = np.sin(np.arange(em.n_faces * d2, dtype=float) * 0.013)
    uhat = np.asfortranarray(core.gather_traces(em, d2, uh))
    return em, t, fields, tau, uhat


def CONFIGS_C2_KAPPA():
    from paper_1305_1489_b200.configs import CONFIGS
    return CONFIGS["C2"].problem.kappa


def cpu_step_seconds(work, nthreads: int, chunk: int = 1024) -> float:
    from oracle import core
    em, t, (kap, c, f), tau, uhat = work
    secs, _ = core.time_pipeline_chunked(em, t, kap, c, f, tau, uhat, nthreads, chunk)
    return secs


def faithful_sample(cfg, nthreads: int, layers: int = 2):
    """Reference-faithful threading (study.cpp:19-31: build + local_blocks on one
    thread, condense + recover on nthreads) on the first `layers` cell layers."""
    from oracle import core
    em, t, (kap, c, f), tau, uhat = oracle_workload(cfg, layers)
    stages = core.time_pipeline(em, t, kap, c, f, tau, uhat, nthreads)
    return em.n_elements / sum(stages[:4]), em.n_elements, stages[:4]


def cpu_baseline_line(cfg, nthreads: int):
    work = oracle_workload(cfg)
    ne = work[0].n_elements
    secs = cpu_step_seconds(work, nthreads)
    from oracle import NATIVE
    line = {"value": ne / secs, "unit": "elements/s", "cores": nthreads, "kind": "port",
            "sample": f"{cfg.name}: the whole {cfg.n}^3 mesh ({ne} tets), one pass, every stage of the reference "
                      f"path over 1024-element chunks on {nthreads} threads (all-cores mode, SURVEY §8(d))",
            "seconds": secs, "march_native": bool(NATIVE)}
    try:
        fv, fne, stages = faithful_sample(cfg, nthreads)
        line["faithful_value"] = fv
        line["faithful_sample"] = (f"first 2 of {cfg.n} cell layers ({fne} tets): build + local_blocks 1 thread, "
                                   f"condense + recover {nthreads} threads (study.cpp:19-31); "
                                   f"stages s={[round(x, 3) for x in stages]}")
    except Exception as exc:  # informative only
        line["faithful_value"] = None
        line["faithful_error"] = repr(exc)[:200]
    return line


def run_reference(args):
    os.environ["HDG_ORACLE_NATIVE"] = "1"   # build/import the -march=native oracle in this process
    from paper_1305_1489_b200.configs import CONFIGS
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    nthreads = os.cpu_count() or 1
    work = oracle_workload(cfg)
    from oracle import NATIVE
    ne = work[0].n_elements
    secs = []
    for i in range(args.warmup + args.steps):
        s = cpu_step_seconds(work, nthreads)
        if i >= args.warmup:
            secs.append(s)
    tot = float(sum(secs))
    v = len(secs) * ne / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "elements/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / len(secs), "higher_is_better": True, "scaling": args.split,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, world, args.split),
            "cpu_baseline": {"value": v, "unit": "elements/s", "cores": nthreads, "kind": "port",
                             "march_native": bool(NATIVE),
                             "sample": f"{cfg.name}: the whole {cfg.n}^3 mesh ({ne} tets; at N > 1 weak, one GPU's "
                                       f"slab) per step, every stage of "
                                       f"the reference path (build_element_matrices -> local_blocks -> condense -> "
                                       f"local_recover) over 1024-element chunks on {nthreads} threads; "
                                       f"lambda gathered outside the timed region"},
            "e2e": {"value": v, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "native_libs": mapped_native_libs()}
    print(json.dumps(line), flush=True)


def mapped_native_libs():
    """Repo-built shared objects mapped into this process (the reference arm must
    show only the oracle's)."""
    try:
        with open("/proc/self/maps") as fh:
            paths = {ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so") and ROOT in ln}
        return sorted(os.path.relpath(p, ROOT) for p in paths)
    except OSError:
        return None


def workload_config(cfg, world: int, split: str = "weak") -> dict:
    n = cfg.n
    if split == "weak":
        box = f"{n}x{n}x{n * world}"
        per = cfg.nelt
    else:
        box = f"{n}x{n}x{n}"
        per = cfg.nelt // world
    return {"workload": f"{cfg.name}: k={cfg.k}, {box} Kuhn box, {per} tets/GPU ({cfg.note})",
            "k": cfg.k, "tets_per_gpu": per, "parallelism": f"z-slabs x{world} ({split})",
            "l2": "flushed (512 MB write) between timed steps; per-step working set > 1 GB"}


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1305_1489_b200 import partition
    from paper_1305_1489_b200.configs import CONFIGS
    from paper_1305_1489_b200.engine import Engine, Field, HostMesh, LocalSolution, dim2, dim3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    prob = cfg.problem
    k = cfg.k
    n = cfg.n
    t_setup = time.perf_counter()
    # weak: rank r owns z-slab r of an n x n x (n * world) box (fixed work per
    # GPU); strong: the config's own n^3 mesh split into world z-slabs
    # (BASELINE C5: "split into contiguous z-slabs over 1/2/4/8 B200")
    nz = n * world if args.split == "weak" else n
    if args.split == "strong" and n % world:
        raise SystemExit(f"--split strong needs {world} to divide the {n} cell layers")
    mesh = HostMesh.box(n, n, nz, bc=prob.bc, perturb=cfg.perturb, seed=cfg.seed)
    sl = partition.slab(mesh, rank, world)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    eng = Engine(local, stream)
    eng.set_degree(k)
    if cfg.postprocess:
        eng.set_postprocess_rule()
    dims = eng.dims
    d3, d2, nq = dims["d3"], dims["d2"], dims["nq"]
    with torch.cuda.stream(stream):
        dm = partition.upload_slab(sl, dev)
        nelt = dm.nelt
        g = eng.geometry(dm, 1.0)
        if cfg.upwind_beta:
            tau = eng.upwind_tau(g, cfg.upwind_beta)
        else:
            tau = cfg.tau
        kap, cc, ff = Field.program(prob.kappa), Field.program(prob.c), Field.program(prob.f)
        cs = eng.alloc_condensed(nelt)
        work = eng.work_buffer(nelt)
        ls = LocalSolution(*(torch.empty(nelt, d3, dtype=torch.float64, device=dev) for _ in range(4)))
        ustar = torch.empty(nelt, dims["d3_post"], dtype=torch.float64, device=dev) if cfg.postprocess else None
        # lambda: a smooth deterministic skeleton vector (values do not change the cost)
        uhat = torch.sin(torch.arange(dm.nfc * d2, dtype=torch.float64, device=dev) * 0.013)
        flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    stream.synchronize()
    t_setup = time.perf_counter() - t_setup

    conv_out = None
    if cfg.upwind_beta:  # C4: the convection block (convdiff.cpp:5-28) is part of the step
        m_ = 4 * d2
        conv_out = tuple(torch.empty(nelt * a, dtype=torch.float64, device=dev) for a in (d3 * d3, m_ * d3, m_ * m_))

    def step():
        eng.geometry(dm, tau, out=g)
        eng.build_condense(g, kap, cc, ff, out=cs, work=work, check=False)
        eng.recover(g, dm, cs, uhat, out=ls)
        if cfg.postprocess:
            eng.postprocess_star(g, kap, ls, out=ustar)
        if conv_out is not None:
            eng.convection_bilinear_matrices(g, cfg.upwind_beta, out=conv_out)

    # geometry 2 (face areas, per element); build_condense 5 (status reset, tau
    # check, K2, K3, rescue screen); recover 1; postprocess 1 (+1 kappa sampler)
    launches_per_step = 2 + 5 + 1 + (2 if cfg.postprocess else 0) + (1 if cfg.upwind_beta else 0)
    eng.set_timing(True)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        stream.synchronize()
        eng.stage_times()
        # singular check once (outside the timed region)
        eng.build_condense(g, kap, cc, ff, out=cs, work=work, check=True)
        eng.stage_times()
        eng.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        stage_acc = {}
        # the step as one CUDA graph (its 8-10 launches replayed without host
        # gaps; launch-bound configs such as C1 gain most); per-kernel times
        # come from eager steps with stage events
        graph = None
        if not args.no_graph:
            try:
                eng.set_timing(False)
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=stream):
                    step()
                gr.replay()
                stream.synchronize()
                graph = gr
            except Exception as exc:  # eager timing instead
                print(f"# CUDA graph capture failed ({exc!r:.120}); timing eager launches", file=sys.stderr)
                graph = None
            finally:
                eng.set_timing(True)
                torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            for i in range(args.steps):
                flush.zero_()
                ev[i][0].record(stream)
                if graph is not None:
                    graph.replay()
                else:
                    step()
                ev[i][1].record(stream)
                if graph is None:
                    for kname, v in eng.stage_times().items():   # waits for this step
                        stage_acc.setdefault(kname, []).append(v)
                else:
                    ev[i][1].synchronize()
        torch.cuda.synchronize()
        if graph is not None:  # per-kernel stage times: eager steps (not the timed ones)
            c_graph = cs.C.clone()
            for _ in range(min(args.steps, 5)):
                flush.zero_()
                step()
                for kname, v in eng.stage_times().items():
                    stage_acc.setdefault(kname, []).append(v)
            torch.cuda.synchronize()
            # the replayed graph and the eager launches compute the same step, bit for bit
            assert torch.equal(c_graph, cs.C), "CUDA graph replay and eager step differ"
            del c_graph
        if world > 1:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    value = world * nelt / (ms_per_step / 1e3)
    stage_ms = {kname: float(np.mean(v)) for kname, v in stage_acc.items()}

    # sanity: outputs finite
    assert torch.isfinite(cs.C).all() and torch.isfinite(ls.u).all(), "non-finite outputs"

    # ------------------------------------------- K4 scatter + slab exchange
    # Reported beside the step ("K4 and the NCCL exchange are
    # reported separately"): slab-local CSR values + b, then the interface
    # faces' diagonal blocks and b summed with the neighbour slabs.
    scatter_info = None
    if not args.no_scatter:
        from paper_1305_1489_b200.distributed import NativeSlabExchange
        fb, nb, slt = partition.slab_pattern(sl)
        with torch.cuda.stream(stream):
            pat = eng.pattern_from_arrays(fb, nb, slt)
            sysH = eng.assemble(dm, pat, cs)
            # the engine's own exchange: C-ABI plan, device gather/add, grouped
            # ncclSend/ncclRecv per neighbour on the engine stream
            ex = NativeSlabExchange(eng, sl, fb, nb, d2)
            if world > 1:
                ex.init_comm(rank, world)
            stream.synchronize()
            if world > 1:
                dist.barrier()
            sc_ms, ex_ms = [], []
            for _ in range(max(1, min(args.steps, 5))):
                a0, a1, a2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                a0.record(stream)
                eng.assemble(dm, pat, cs, out=sysH)
                a1.record(stream)
                if world > 1:
                    ex.exchange(sysH.vals, sysH.b)
                a2.record(stream)
                a2.synchronize()
                sc_ms.append(a0.elapsed_time(a1))
                ex_ms.append(a1.elapsed_time(a2))
        eng.stage_times()
        sc_med, ex_med = float(np.median(sc_ms)), float(np.median(ex_ms))
        if world > 1:
            t = torch.tensor([sc_med + ex_med], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            both = float(t.item())
        else:
            both = sc_med + ex_med
        scatter_info = {"scatter_ms": sc_med, "exchange_ms": ex_med,
                        "nnz": int(sysH.vals.numel()), "interface_faces": int(len(sl.interface)),
                        "exchange_bytes": int(sum(ex.entries) * 8),
                        "exchange": "hdg_b200_exchange_interface (NCCL grouped send/recv)" if world > 1 else "none (1 rank)",
                        "with_scatter": {"value": world * nelt / ((ms_per_step + both) / 1e3), "unit": "elements/s",
                                         "ms_per_step": ms_per_step + both,
                                         "note": "step + K4 scatter + interface exchange, max over ranks"},
                        # C and Cf read once, every CSR value and b entry written once
                        "scatter_bytes": 8.0 * ((4 * d2) * (4 * d2 + 1) * nelt + sysH.vals.numel() + sysH.b.numel()),
                        }
        scatter_info["scatter_hbm_gbs"] = scatter_info["scatter_bytes"] / (sc_med / 1e3) / 1e9
        del sysH, pat

    # ------------------------------------------------------- SAMPLED leg
    # The reference's own API shape (ScalarField callbacks, coefficient.hpp:
    # 13-14): the caller samples its callbacks at the device's physical nodes
    # (hdg_b200_quad_points; here torch expressions of the same fields) and
    # passes HDG_FIELD_SAMPLED arrays, which K2 reads (3 nq 8 B per element).
    # Timed: geometry, quad points, the caller's callbacks, build+condense,
    # recover.
    sampled_info = None
    if not args.no_sampled and not cfg.upwind_beta:
        import math
        env = {"sin": torch.sin, "cos": torch.cos, "exp": torch.exp, "sqrt": torch.sqrt, "abs": torch.abs,
               "pi": math.pi, "lt": lambda a, b: (a < b).double(), "pow": torch.pow}
        cb = [compile(e, "<field>", "eval") for e in (prob.kappa, prob.c, prob.f)]

        def callbacks(X, Y, Z):
            loc = {"x": X, "y": Y, "z": Z}
            return [torch.as_tensor(eval(c_, env, loc), dtype=torch.float64, device=dev).expand_as(X).contiguous()
                    for c_ in cb]

        def sampled_step():
            eng.geometry(dm, tau, out=g)
            X, Y, Z = eng.quad_points(g)
            sk, sc_, sf = callbacks(X, Y, Z)
            eng.build_condense(g, Field.sampled(sk), Field.sampled(sc_), Field.sampled(sf), out=cs, work=work,
                               check=False)
            eng.recover(g, dm, cs, uhat, out=ls)

        with torch.cuda.stream(stream):
            for _ in range(2):
                sampled_step()
            sms = []
            for _ in range(max(1, min(args.steps, 5))):
                flush.zero_()
                b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                b0.record(stream)
                sampled_step()
                b1.record(stream)
                b1.synchronize()
                sms.append(b0.elapsed_time(b1))
        eng.stage_times()
        smed = float(np.median(sms))
        if world > 1:
            t = torch.tensor([smed], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            smed = float(t.item())
        sampled_info = {"value": world * nelt / (smed / 1e3), "unit": "elements/s", "ms_per_step": smed,
                        "path": "hdg_b200_quad_points -> caller's torch callbacks at the nodes -> HDG_FIELD_SAMPLED "
                                "build_condense -> recover",
                        "sample_bytes_per_element": 3 * nq * 8}

    # ---------------------------------------------------------------- e2e
    # Through the public API with HOST buffers: H2D of the step's inputs (mesh
    # arrays + lambda, pinned), the step, D2H of its results (C, Cf, q, u).
    # The element range is processed in E2E_CHUNKS contiguous chunks (each its
    # own DeviceMesh/Geometry; the outputs are contiguous slices of the global
    # Batch3/column-major arrays), and the D2H of chunk i runs on a copy stream
    # while chunk i+1 computes: the step is PCIe-bound (2.7 GB of C at C2), so
    # this overlap is the end-to-end schedule a user of the API would run.
    from paper_1305_1489_b200.engine import CondensedSystem, DeviceMesh, Geometry
    E2E_CHUNKS = 4
    bounds = [round(i * nelt / E2E_CHUNKS) for i in range(E2E_CHUNKS + 1)]
    m = 4 * d2
    nf = dims["factors"]
    host_shared = [t.cpu().pin_memory() for t in (dm.coords, dm.faces, uhat)]
    dev_shared = [dm.coords, dm.faces, uhat]
    host_el = dm.elements.cpu()
    host_fb = dm.facebyele.cpu()
    chunks = []
    for i in range(E2E_CHUNKS):
        k0, k1 = bounds[i], bounds[i + 1]
        nc = k1 - k0
        h_el = host_el[:, k0:k1].contiguous().pin_memory()
        h_fb = host_fb[:, k0:k1].contiguous().pin_memory()
        dmc = DeviceMesh(dm.nver, nc, dm.nfc, dm.coords, dm.elements[:, k0:k1].contiguous(), dm.faces,
                         dm.facebyele[:, k0:k1].contiguous(), dm.facetype, dm.ndir, dm.nneu)
        gc = eng.geometry(dmc, 1.0)
        csc = CondensedSystem(cs.C[k0 * m * m:k1 * m * m], cs.Cf[k0 * m:k1 * m], cs.factors[k0 * nf:k1 * nf], m)
        lsc = LocalSolution(ls.qx[k0:k1], ls.qy[k0:k1], ls.qz[k0:k1], ls.u[k0:k1])
        usc = ustar[k0:k1] if cfg.postprocess else None
        outs_c = [csc.C, csc.Cf, lsc.qx, lsc.qy, lsc.qz, lsc.u] + ([usc] if cfg.postprocess else [])
        host_c = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs_c]
        chunks.append(dict(h_in=[h_el, h_fb], d_in=[dmc.elements, dmc.facebyele], dm=dmc, g=gc, cs=csc,
                           ls=lsc, us=usc, outs=outs_c, host=host_c, work=eng.work_buffer(nc),
                           ev=torch.cuda.Event()))
    h2d = sum(t.numel() * t.element_size() for t in host_shared) + \
        sum(t.numel() * t.element_size() for c in chunks for t in c["h_in"])
    d2h = sum(t.numel() * t.element_size() for c in chunks for t in c["host"])
    copy_stream = torch.cuda.Stream(dev)
    e2e_steps = max(1, min(args.steps, 5))

    def e2e_step():
        for h, d in zip(host_shared, dev_shared):
            d.copy_(h, non_blocking=True)
        for c in chunks:
            for h, d in zip(c["h_in"], c["d_in"]):
                d.copy_(h, non_blocking=True)
            eng.geometry(c["dm"], tau, out=c["g"])
            eng.build_condense(c["g"], kap, cc, ff, out=c["cs"], work=c["work"], check=False)
            eng.recover(c["g"], c["dm"], c["cs"], uhat, out=c["ls"])
            if cfg.postprocess:
                eng.postprocess_star(c["g"], kap, c["ls"], out=c["us"])
            c["ev"].record(stream)
            copy_stream.wait_event(c["ev"])
            with torch.cuda.stream(copy_stream):
                for h, d in zip(c["host"], c["outs"]):
                    h.copy_(d, non_blocking=True)
        stream.wait_stream(copy_stream)

    with torch.cuda.stream(stream):
        e2e_step()  # warm-up (chunk-sized work buffers, JIT cache)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(stream)
        e1.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    eng.set_timing(False)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    hbm_peak, hbm_src = load_peaks()
    k3_ms = stage_ms.get("condense", float("nan"))
    achieved = k3_flops(k) * nelt / (k3_ms / 1e3) / 1e12
    kname3 = f"condense6_kernel<{k}" if k in (2, 3) else (f"condense2_kernel<{k}>" if k <= 1 else
                                                          f"condense5_kernel<{k}>")
    traffic, traffic_src = ncu_traffic(kname3)
    roof = {"kernel": (kname3 + (", warps>" if k in (2, 3) else "")) + " (K3)", "bound": "tensor", "achieved": achieved,
            "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
            "traffic": traffic if cfg.name == "C2" and world == 1 else None,
            "traffic_source": traffic_src,
            "peak_source": FP64_PEAK_SOURCE, "flops_per_element": k3_flops(k),
            "flops_per_launch": k3_flops(k) * nelt, "launch_ms": k3_ms,
            "pipe": "fp64 (DMMA mma.sync m8n8k4)"}
    if k == 3:
        # Explains frac (not a second claim): how busy the fp64 pipe is with the
        # instructions K3 v6 executes per element (ncu instruction counts of the
        # committed capture: K3_DMMA_PER_ELT DMMA.8x8x4 at one per 16 sub-partition
        # cycles, K3_FP64_ALU_PER_ELT DFMA/DMUL/DADD at one per 2), over the measured launch time at the
        # sampled SM clock. Padding (d3 = 20 in 24-wide tiles) and the sweeps'
        # DFMAs are pipe time that frac, counted on algorithmic flops, leaves out.
        sm_mhz = (clk.summary() or {}).get("sm_mhz") or 1965.0
        pipe_cycles = K3_DMMA_PER_ELT * 16 + K3_FP64_ALU_PER_ELT * 2
        roof["fp64_pipe"] = {"dmma_per_element": K3_DMMA_PER_ELT, "fp64_alu_per_element": K3_FP64_ALU_PER_ELT,
                             "pipe_cycles_per_element": pipe_cycles,
                             "busy_frac": pipe_cycles * nelt / (c_sms(dev) * 4 * (k3_ms / 1e3) * sm_mhz * 1e6),
                             "source": "profiles/r02f_ncu_k3v6_c2.txt (executed instruction counts)"}
    # SURVEY §8(d) compulsory HBM bytes of the whole step (mesh + geometry for
    # build and for recover, coefficient samples when SAMPLED, C + Cf written,
    # lambda gathered, q + u written); caches and intermediates are not
    # algorithmic. The fields here are PROGRAMs evaluated at the nodes (no sample reads).
    alg = step_algorithmic_bytes(k, nq, sampled=False) * nelt
    step_dram, step_src = ncu_step_traffic()
    traffic_info = {"algorithmic_bytes": alg, "algorithmic_bytes_per_element": alg / nelt,
                    "dram_bytes": step_dram if cfg.name == "C2" and world == 1 else None, "source": step_src,
                    "dram_over_algorithmic": (step_dram / alg) if (step_dram and cfg.name == "C2" and world == 1) else None,
                    "algorithmic_gbs": alg / (ms_per_step / 1e3) / 1e9, "hbm_peak_gbs": hbm_peak}
    kern = {}
    for kname, v in stage_ms.items():
        kern[kname] = {"ms": v}
    if "node_build" in stage_ms:
        kern["node_build"]["tflops"] = k2_flops(k, nq) * nelt / (stage_ms["node_build"] / 1e3) / 1e12
    if "condense" in stage_ms:
        kern["condense"]["tflops"] = achieved
    if "recover" in stage_ms:
        rb = 8.0 * (dims["factors"] + 4 * d2 + 30 + 4 * d3)
        kern["recover"]["hbm_gbs"] = rb * nelt / (stage_ms["recover"] / 1e3) / 1e9
        kern["recover"]["hbm_frac"] = kern["recover"]["hbm_gbs"] / hbm_peak
    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.split,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (closed-form fields at the nodes, BASELINE configs)",
        "config": workload_config(cfg, world, args.split),
        "roofline": roof,
        "traffic": traffic_info,
        "kernels_ms": kern,
        "e2e": {"value": world * nelt / (e2e_ms / 1e3), "unit": "elements/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "chunks": E2E_CHUNKS,
                "path": "pinned host mesh+lambda -> C ABI step in 4 element chunks, D2H of chunk i overlapped with chunk i+1 -> pinned host C, Cf, q, u"},
        "scatter": scatter_info,
        "sampled_fields": sampled_info,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "setup_s": t_setup,
    }
    line["config"]["step_launch"] = ("one CUDA graph replay per step (the captured launches)" if graph is not None
                                     else "eager launches")
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_line(cfg, os.cpu_count() or 1)
            line["speedup_vs_cpu_baseline"] = value / line["cpu_baseline"]["value"]
        except Exception as exc:  # the CPU leg must not sink the GPU line
            line["cpu_baseline"] = {"value": None, "error": repr(exc)[:200]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--split", default="weak", choices=["weak", "strong"],
                    help="multi-GPU: weak = an n^3 slab per GPU, strong = the config's n^3 mesh split in z-slabs")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the step as eager launches instead of one CUDA graph replay")
    ap.add_argument("--no-sampled", action="store_true", help="skip the HDG_FIELD_SAMPLED leg")
    ap.add_argument("--no-scatter", action="store_true",
                    help="skip the separately reported K4 scatter + interface exchange timing")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: L(θ) evaluations/s (H-assemble + H-Cholesky + logdet + solve).

Workload (BASELINE.json configs[2], "C3"): n = 262144 points on a 512x512
jittered grid (seed 1), θ = (σ²=1.5, ℓ=0.05, ν=1.0 general-ν Bessel path,
τ²=0.01), Z iid N(0,1) (seed 1 ^ 0x517cc1b727220a95), leaf 128, η = 2,
ε = 1e-6, H-Cholesky.  One step = one full L(θ): cluster tree + block tree
(K1, K2), assembly (K3 dense leaves, K4 ACA, K5 recompression), H-Cholesky
(K6-K9), log-determinant + forward solve (K10, K11).

  value : device-resident coordinates and Z (torch tensors in HBM) through
          hmgp_geometry_build_device + hmgp_loglik_geom; CUDA events on the
          library stream; max over ranks.
  e2e   : the public API call hmgp_loglik with HOST buffers (H2D of coords + Z and
          D2H of the result inside the timed region).
  Multi-GPU (``--gpus N``: under torchrun the ranks come from the environment,
  otherwise this script spawns N ranks itself): one L(θ) does not shard
  (SURVEY.md §8e), an MLE θ-sweep does — rank r evaluates its own θ of a C3-sized
  sweep (ℓ nudged per rank), K steps each, and ONE NCCL all-gather
  (hmgp_sweep_gather, the C ABI's own communicator) collects the N values inside
  the timed region; value = N*K / max-over-ranks time, weak scaling.  The
  per-N ``extras`` shard the C4 θ-grid subset (ν-major), the C4 kriging points
  (argmax θ of the sweep) and the C2 leaf assembly over the same ranks.

``--impl reference`` times the CPU restatement of the reference (oracle/, the
reference itself cannot be built here: Eigen is absent) on the host cores: one
bounded sample (n = 65536 at the C3 density/θ/leaf/ε, ~4 min) scaled to n = 262144
by the ratio of the same code's committed full-size and n = 65536 timings
(tests/golden/oracle_timing_c3.json) — a 4x step in n, not a fitted exponent.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading

import numpy as np
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# 32 hardware work queues for the task-flow factorization's streams (before any
# CUDA context exists in this process)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, ROOT)

C3 = dict(g=512, leaf=128, eps=1e-6, theta=(1.5, 0.05, 1.0, 0.01), form="cholesky")
WORKLOAD = ("C3: n=262144 2D jittered 512x512 grid, Matern theta=(1.5,0.05,1.0,0.01) general-nu, "
            "Z iid N(0,1), leaf 128, eta 2, eps 1e-6, H-Cholesky")
METRIC = "L(θ) evals/s (H-assemble+H-Cholesky+logdet+solve) at n=256K; FP64 roofline %"
SEED = 1
Z_SEED = SEED ^ 0x517CC1B727220A95


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for k, nm in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                pass
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# --------------------------------------------------------------------------
def _bcast_bytes(dist, device):
    """Launcher-side hand-over of the C ABI's ncclUniqueId (rank 0 -> all)."""
    import torch

    def bcast(raw):
        t = torch.zeros(128, dtype=torch.uint8, device=device)
        if raw is not None:
            t.copy_(torch.tensor(list(raw), dtype=torch.uint8))
        dist.broadcast(t, 0)
        return bytes(t.cpu().tolist())
    return bcast


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2104_07146_b200 as hm
    from paper_2104_07146_b200 import _lib
    from paper_2104_07146_b200 import sweep as sw

    ws, rank, lrank = dist_env()
    torch.cuda.set_device(lrank)
    dev = torch.device("cuda", lrank)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = hm.Context(lrank)
    _lib.hmgp_ctx_stream.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    _lib.hmgp_last_phases.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int]
    _lib.hmgp_work_counters.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int]
    _lib.hmgp_fp64_peak.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    _lib.hmgp_set_flop_counting.argtypes = [C.c_int]
    sp = C.c_void_p()
    hm._chk(_lib.hmgp_ctx_stream(ctx.h, C.byref(sp)))
    stream = torch.cuda.ExternalStream(sp.value, device=dev)
    # the C ABI's own NCCL communicator for the result gathers (world 1: no NCCL)
    comm = sw.Comm(ctx, rank, ws, _bcast_bytes(dist, dev) if ws > 1 else None)

    cfgd = dict(C3)
    if args.small:  # quick functional runs (not a bench line)
        cfgd.update(g=128)
    g = cfgd["g"]
    n = g * g
    x = hm.jittered_grid(g, SEED)
    z = hm.normals(n, Z_SEED)
    # the θ of this rank's share of a C3-sized sweep (rank 0: the C3 θ itself)
    sweep_thetas = np.array([[cfgd["theta"][0], cfgd["theta"][1] * (1.0 + 1e-3 * r), cfgd["theta"][2],
                              cfgd["theta"][3]] for r in range(ws)])
    theta = hm.Matern(*sweep_thetas[rank])
    cfg = hm.HConfig(leaf_size=cfgd["leaf"], rank=hm.RankControl.fixed_accuracy(cfgd["eps"]),
                     form=cfgd["form"]).c()
    # device-resident inputs (torch = plumbing only)
    dx = torch.from_numpy(x).to(dev)
    dz = torch.from_numpy(z).to(dev)
    torch.cuda.synchronize()
    res = hm._LogLik()
    my_idx = np.array([rank], dtype=np.int32)
    gathered = {}

    def step_device():
        gh = C.c_void_p()
        hm._chk(_lib.hmgp_geometry_build_device(ctx.h, C.c_void_p(dx.data_ptr()), n, 2,
                                                cfgd["leaf"], 2.0, C.byref(gh)))
        try:
            hm._chk(_lib.hmgp_loglik_geom(ctx.h, gh, C.c_void_p(dz.data_ptr()), C.byref(theta),
                                          C.byref(cfg), C.byref(res)))
        finally:
            _lib.hmgp_geometry_destroy(gh)

    def step_e2e():
        hm._chk(_lib.hmgp_loglik(ctx.h, x.ctypes.data_as(hm._dp), n, 2, z.ctypes.data_as(hm._dp),
                                 C.byref(theta), C.byref(cfg), C.byref(res)))

    def gather():  # the sweep's only collective: N result rows
        rows = (hm._LogLik * 1)(res)
        gathered["table"] = sw.gather_c(ctx, comm, my_idx, rows, ws)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, k):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(k):
            fn()
        gather()
        e1.record(stream)
        e1.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if ws > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # untimed counting pass (algorithmic work of one step) + FP64 peak
    w = (C.c_double * 10)()
    _lib.hmgp_work_counters(w, 10, 1)
    _lib.hmgp_set_flop_counting(1)
    step_device()
    _lib.hmgp_set_flop_counting(0)
    _lib.hmgp_work_counters(w, 10, 1)
    work = dict(zip(["dense_entries", "aca_entries", "kernel_flops", "gemm_flops", "trsm_flops",
                     "leaf_flops", "trunc_flops", "trunc_items", "arena_peak_bytes", "factor_attempts"], list(w)))
    peak = C.c_double()
    hm._chk(_lib.hmgp_fp64_peak(ctx.h, C.byref(peak)))
    fp64_peak = peak.value

    for _ in range(args.warmup):
        step_device()
    launches0 = ctx.launches()
    clk = Clocks(lrank)
    clk.start()
    ms = timed(step_device, args.steps)
    clocks = clk.stop()
    launches = (ctx.launches() - launches0) // max(1, args.steps)
    loglik = res.loglik
    ph = (C.c_double * 10)()
    _lib.hmgp_last_phases(ctx.h, ph, 10)
    phases = dict(zip(["start", "geometry", "dense_K3", "aca_K4K5", "layout", "factor_K6K9",
                       "logdet_K11", "fwd_solve_K10", "bwd", "cross_K12"], list(ph)))
    # e2e through the public API with host buffers
    step_e2e()
    ms_e2e = timed(step_e2e, max(1, args.steps))

    line = None
    if rank == 0:
        value = ws * args.steps / (ms / 1e3)
        e2e_value = ws * max(1, args.steps) / (ms_e2e / 1e3)
        peaks = measured_peaks()
        # dominant kernel family of the step and its roofline
        fam = {
            "factor_K6K9": (work["gemm_flops"] + work["trsm_flops"] + work["leaf_flops"]
                            + work["trunc_flops"], phases["factor_K6K9"]),
            "dense_K3": (work["kernel_flops"], phases["dense_K3"]),
        }
        dom = max(fam, key=lambda k: fam[k][1])
        flops, pms = fam[dom]
        achieved = flops / (pms / 1e3) / 1e12 if pms > 0 else 0.0
        roofline = {"bound": "fp64", "kernel": dom, "achieved": achieved, "peak": fp64_peak,
                    "unit": "TFLOP/s", "frac": achieved / fp64_peak if fp64_peak else None,
                    "traffic": None, "peak_source": "measured FP64 FMA-chain microbenchmark "
                    "(hmgp_fp64_peak) on this B200; MEASURED_PEAKS.json has no FP64 entry",
                    "share_of_step": pms / (ms / args.steps),
                    "algorithmic_flops_per_launch": flops}
        # Matérn assembly (K3 dense near-field leaves, general-ν Bessel path at C3):
        # flop-model work of the untimed counting pass over the live K3 phase time
        k3_ms = phases["dense_K3"]
        k3_ach = work["kernel_flops"] / (k3_ms / 1e3) / 1e12 if k3_ms > 0 else 0.0
        roofline_asm = {"bound": "fp64", "kernel": "dense_K3 (k_dense_leaves)", "achieved": k3_ach,
                        "peak": fp64_peak, "unit": "TFLOP/s",
                        "frac": k3_ach / fp64_peak if fp64_peak else None,
                        "algorithmic_flops_per_launch": work["kernel_flops"],
                        "entries_per_launch": work["dense_entries"],
                        "flop_model": "per-entry Temme/Steed iteration path, exp/log/sin/sinh/cosh = 20, pow = 45"}
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded jittered grid + AS241 normals, simgen conventions)",
            "config": bench_config(args, n, cfgd, ws),
            "loglik": loglik, "phases_ms_last_step": phases, "work_per_step": work,
            "clocks": clocks, "gpu_launches": int(launches),
            "e2e": {"value": e2e_value, "unit": "evals/s",
                    "h2d_bytes_per_step": 8 * n * 2 + 8 * n, "d2h_bytes_per_step": C.sizeof(res)},
            "roofline": roofline,
            "roofline_assembly": roofline_asm,
            "hbm_peak_gbs": peaks.get("hbm_gbs"),
        }
        if ws > 1:
            line["sweep_loglik"] = gathered["table"][:, 0].tolist()
            line["collective"] = "one ncclAllGather of N result rows per timed region (hmgp_sweep_gather)"
    if not args.no_extras and not args.small:
        ex = extras(hm, _lib, ctx, stream, comm, rank, ws, peaks=measured_peaks(), c3_batch=args.c3_batch,
                    step_phases=phases)
        if line is not None:
            line["extras"] = ex
    if line is not None:
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    comm.close()
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def bench_config(args, n, cfgd, ws):
    return {"workload": WORKLOAD if not args.small else "small functional run g=128",
            "n": n, "leaf_size": cfgd["leaf"], "eta": 2.0, "eps": cfgd["eps"],
            "form": cfgd["form"],
            "parallelism": "1 GPU" if ws == 1 else f"theta-sweep shards x{ws} (one L(theta) per rank per step)",
            "l2": "inputs larger than L2 (>2 GB near-field payload per step)"}


def extras(hm, _lib, ctx, stream, comm, rank, ws, peaks, c3_batch=False, step_phases=None):
    """Other BASELINE configs, measured once each (device events on the library
    stream, max over ranks): C3 θ-batch, solve / matvec HBM rooflines, C2
    assembly (sharded over the ranks), the C4 θ-grid subset sharded ν-major with
    ONE result gather, and C4 kriging with the argmax θ sharded over the ranks."""
    import torch
    import torch.distributed as dist
    from paper_2104_07146_b200 import sweep as sw
    out = {}
    dev = torch.device("cuda", ctx.device)

    def dev_ms(fn):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        r = fn()
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        if ws > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, r

    hbm = peaks.get("hbm_gbs") or 6546.9
    xc3 = hm.jittered_grid(C3["g"], SEED)
    zc3h = hm.normals(C3["g"] ** 2, Z_SEED)
    gc3 = hm.Geometry(xc3, C3["leaf"], 2.0, ctx=ctx)
    cfg3 = hm.HConfig(leaf_size=C3["leaf"], rank=hm.RankControl.fixed_accuracy(C3["eps"]), form=C3["form"])
    if rank == 0:
        # HBM-bound kernels at C3: H-matvec (reads the H-matrix payload once) and the
        # forward solve K10 (reads the factor payload once).  Algorithmic bytes =
        # payload bytes + the vectors; timed through the host-buffer C ABI call
        # (2 MB of vector copies inside the timed region, noted).
        h3 = hm.assemble(gc3, list(C3["theta"]), hm.RankControl.fixed_accuracy(C3["eps"]))
        hb = h3.stats()["bytes"]
        dzv = torch.from_numpy(zc3h).to(dev)
        dyv = torch.empty_like(dzv)
        mv = lambda: hm._chk(_lib.hmgp_hmat_matvec_device(ctx.h, h3.h, C.c_void_p(dzv.data_ptr()),  # noqa: E731
                                                          C.c_void_p(dyv.data_ptr())))
        mv()
        ms_mv, _ = dev_ms(lambda: [mv() for _ in range(5)])
        ms_mv /= 5.0
        f3 = hm.factorize(h3, C3["eps"], C3["form"])
        fb = f3.info["storage_bytes"]
        f3.solve_lower(zc3h)
        ms_sl, _ = dev_ms(lambda: f3.solve_lower(zc3h))
        nvec = 8.0 * C3["g"] ** 2
        out["roofline_matvec"] = {"bound": "hbm", "kernel": "H-matvec (k_mv_leaf + k_mv_chunk_* + k_mv_gather)",
                                  "ms": ms_mv, "algorithmic_bytes": hb + 2 * nvec,
                                  "achieved": (hb + 2 * nvec) / ms_mv / 1e6,
                                  "peak": hbm, "unit": "GB/s", "frac": (hb + 2 * nvec) / ms_mv / 1e6 / hbm,
                                  "traffic": 5712027480.0,
                                  "traffic_source": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum over "
                                  "the product's seven kernels (profiles/r2_hbm_kernels_raw.csv): 1.45x the "
                                  "algorithmic bytes - tall low-rank leaves are read twice (dots, then apply), "
                                  "plus the private output segments; the kernels run at 4.2-5.2 TB/s of DRAM",
                                  "note": "device vectors (hmgp_hmat_matvec_device), mean of 5 "
                                  "back-to-back products; payload 4 GB >> L2"}
        # the forward solve of the timed step itself (device events of its K10 phase:
        # gather + sweep + quadratic-form reduction), over this factor's payload bytes
        ms_k10 = (step_phases or {}).get("fwd_solve_K10") or ms_sl
        out["roofline_solve"] = {"bound": "hbm", "kernel": "forward solve K10 (k_solve_sweep)", "ms": ms_k10,
                                 "algorithmic_bytes": fb + 2 * nvec, "achieved": (fb + 2 * nvec) / ms_k10 / 1e6,
                                 "peak": hbm, "unit": "GB/s", "frac": (fb + 2 * nvec) / ms_k10 / 1e6 / hbm,
                                 "traffic": 3986579000.0,
                                 "traffic_source": "ncu --set full of k_solve_sweep (profiles/r2_solve_sweep_raw.csv): "
                                 "3.964 GB read + 22 MB written = 1.01x the algorithmic bytes",
                                 "host_buffer_call_ms": ms_sl,
                                 "note": "K10 phase of the last timed step; bound by its 2048-step dependency "
                                         "chain, not by HBM (DESIGN.md section 6)"}
        del f3, h3
    # C3 θ-throughput: the same n = 262144 problem, 9 θ per rank (ℓ nudged) through
    # hmgp_loglik_sweep on one geometry: θ0 alone sizes the workspace, the other 8 run
    # concurrently on the persistent workers.  (A one-off batch stays on the stream
    # path; long sweeps replay captured CUDA graphs from each worker's third θ on —
    # profiles/r2_exp_graph_batch*.txt.)
    # Opt-in (--c3-batch, ~2 min): one θ needs ~45 GB of device workspace at this size,
    # so at most 3 run concurrently on one B200 and the batch gains little (measured
    # 0.12-0.16 evals/s, profiles/r2_exp_graph_batch_cold_warm.txt); C3-sized sweeps
    # shard over GPUs instead (the headline line with --gpus N).
    if c3_batch:
        th3 = np.array([[C3["theta"][0], C3["theta"][1] * (1.0 + 0.01 * (k + 9 * rank)), C3["theta"][2],
                         C3["theta"][3]] for k in range(9)])
        ms3, (_, v3) = dev_ms(lambda: sw.sweep_host(gc3, zc3h, th3, list(range(9)), cfg3, ctx))
        out["C3_theta_batch"] = {"n": C3["g"] ** 2, "thetas_per_rank": 9, "ms": ms3,
                                 "evals_per_s": 9 * ws / (ms3 / 1e3), "loglik": v3[:, 0].tolist(),
                                 "status": v3[:, 3].tolist(),
                                 "note": "9 θ via hmgp_loglik_sweep: θ0 alone, then 8 on the persistent workers"}
    del gc3
    # C2: assembly only, n = 65536 jittered 256x256, leaf 64, eta 2, eps 1e-7; with N
    # ranks each assembles its cost-balanced leaf range (no collective); the time is
    # the slowest shard's
    x = hm.jittered_grid(256, SEED)
    g = hm.Geometry(x, 64, 2.0, ctx=ctx)
    cnt, na, nd = g.block_counts()
    c2 = {"n": 65536, "leaf": 64, "eps": 1e-7, "blocks": int(cnt), "admissible": int(na), "dense": int(nd),
          "shards": ws}
    w = (C.c_double * 10)()
    rc7 = hm.RankControl.fixed_accuracy(1e-7)
    for nu in (0.5, 1.5, 0.325):
        th = [1.0, 0.1, nu, 0.01]
        asm = (lambda: hm.assemble(g, th, rc7)) if ws == 1 else (lambda: hm.assemble_shard(g, th, rank, ws, rc7))
        asm()  # warm-up
        _lib.hmgp_work_counters(w, 10, 1)
        ms, h = dev_ms(asm)
        _lib.hmgp_work_counters(w, 10, 1)
        ent = torch.tensor([w[0], w[1]], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(ent)
        d_e, a_e = float(ent[0]), float(ent[1])
        c2[f"nu={nu}"] = {"ms": ms, "entries": d_e + a_e, "entries_per_s": (d_e + a_e) / (ms / 1e3),
                          "dense_entries": d_e, "aca_entries": a_e}
        del h
    out["C2_assembly"] = c2
    # C4: n = 65536 training (jittered), Z ~ N(0, C(θ₀)) exact sample, θ₀ = (1, 0.1,
    # 0.5, 0.01) (BASELINE configs[3]) via the device dense sampler (34 GB FP64
    # covariance + POTRF; a data utility, outside every timed region)
    t0 = time.time()
    z = hm.sample_grf(x, [1.0, 0.1, 0.5, 0.01], Z_SEED, ctx=ctx)
    out["C4_data"] = {"z": "sample_grf(theta0=(1,0.1,0.5,0.01), seed 1^0x517cc1b727220a95)",
                      "sample_grf_s": time.time() - t0}
    cfg = hm.HConfig(leaf_size=64, rank=hm.RankControl.fixed_accuracy(1e-7))
    # C4 θ-sweep: 16·N θ of the 512-point grid (every ν and τ², grid σ² / ℓ values
    # around θ₀), sharded ν-major over the ranks (hmgp_sweep_shard), ONE gather
    grid = sw.c4_theta_grid()
    pick = [(s, l) for l in (sw.C4_ELL[3], sw.C4_ELL[2], sw.C4_ELL[4], sw.C4_ELL[1])
            for s in (sw.C4_SIGMA2[3], sw.C4_SIGMA2[4], sw.C4_SIGMA2[2], sw.C4_SIGMA2[5])][: 2 * ws]
    sub = [i for i in range(len(grid)) if (grid[i, 0], grid[i, 1]) in pick]
    sub_thetas = grid[sub]
    mine = sw.shard_c(sub_thetas, rank, ws)

    def run_c4():
        rows, _ = sw.sweep_host(g, z, sub_thetas, list(mine), cfg, ctx)
        return sw.gather_c(ctx, comm, mine, rows, len(sub))
    ms_sw, table = dev_ms(run_c4)
    kbest, th_best, l_best = sw.argmax_theta(sub_thetas, table)
    out["C4_sweep_subset"] = {"n": 65536, "thetas": len(sub), "of_grid": 512, "ms": ms_sw,
                              "evals_per_s": len(sub) / (ms_sw / 1e3),
                              "theta_idx": [int(i) for i in sub], "loglik": table[:, 0].tolist(),
                              "status": table[:, 3].tolist(),
                              "argmax_theta": [float(v) for v in th_best], "argmax_loglik": float(l_best),
                              "shard": "nu-major round-robin (hmgp_sweep_shard), one ncclAllGather"}
    # C4 kriging at m = 10000 uniform test points with the ARGMAX θ of the sweep:
    # every rank factors C̃11 itself and predicts its contiguous slice; one gather
    te = hm.random_locations(10000, SEED + 1)
    lo, hi = sw.predict_ranges(10000, ws)[rank]
    thb = [float(v) for v in th_best]
    hm.predict(x, z, te[:100], thb, cfg, ctx=ctx)  # warm-up

    def run_pred():
        loc = hm.predict(x, z, te[lo:hi], thb, cfg, ctx=ctx).z2_hat
        return sw.predict_gather_c(ctx, comm, loc, 10000)
    ms, pr = dev_ms(run_pred)
    ph = (C.c_double * 10)()
    _lib.hmgp_last_phases(ctx.h, ph, 10)
    out["C4_kriging"] = {"n": 65536, "m": 10000, "theta": thb, "ms": ms,
                         "predictions_per_s": 10000 / (ms / 1e3),
                         "cross_covariance_ms": ph[9],
                         "cross_entries_per_s": (hi - lo) * 65536 / (ph[9] / 1e3) if ph[9] > 0 else None,
                         "factor_ms": ph[5], "pred_checksum": float(np.sum(pr)),
                         "shard": "contiguous m/N slices (hmgp_predict_range), one ncclAllGather"}
    return out


# --------------------------------------------------------------------------
def _oracle_eval(o, g, threads):
    from oracle.oracle import make_config
    x = o.jittered_grid(g, SEED)
    z = o.normals(g * g, Z_SEED)
    cfg = make_config(leaf_size=C3["leaf"], eps=C3["eps"], form=C3["form"], threads=threads)
    t = time.time()
    r = o.loglik(x, z, list(C3["theta"]), cfg)
    return time.time() - t, r


def _timing_fixture():
    with open(os.path.join(ROOT, "tests", "golden", "oracle_timing_c3.json")) as f:
        return json.load(f)


def cpu_baseline(g=96):
    """CPU restatement (oracle, 'port') on the host cores, bounded sample.

    One timed oracle L(θ) at n = g² with the C3 density/θ/leaf/ε, scaled to
    n = 262144 by the MEASURED ratio of the same code's timings on the build box
    (tests/golden/oracle_timing_c3.json: the full C3 run took 1543 s there) —
    not a fitted exponent.  Assembly uses all host threads (hmatrix.cpp:193), the
    factorization one (as the reference)."""
    from oracle.oracle import Oracle
    o = Oracle()
    threads = os.cpu_count() or 1
    fx = _timing_fixture()["seconds"]
    ts, _ = _oracle_eval(o, g, threads)
    ratio = fx["262144"] / fx[str(g * g)]
    t_c3 = ts * ratio
    return {"value": 1.0 / t_c3, "unit": "evals/s", "cores": threads, "kind": "port",
            "sample": (f"one oracle L(θ) at n={g * g} (C3 density/θ/leaf/ε): {ts:.2f}s here; x{ratio:.1f} = the "
                       f"same code's measured n=262144 / n={g * g} time ratio on the build box "
                       f"({fx['262144']:.0f}s / {fx[str(g * g)]:.2f}s, tests/golden/oracle_timing_c3.json) "
                       f"-> {t_c3:.0f}s per C3 eval; assembly on {threads} threads, factorization single-threaded"),
            "sample_seconds": ts, "sample_n": g * g, "scale_ratio": ratio}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    # one bounded sample per run (the requested steps would take hours on the CPU):
    # n = 65536 (a 4x step below C3) unless --ref-g picks another measured size
    t0 = time.time()
    cb = cpu_baseline(g=args.ref_g)
    wall = time.time() - t0
    cfgd = dict(C3)
    line = {"metric": METRIC, "value": cb["value"], "unit": "evals/s", "n_gpus": ws,
            "steps": 1, "warmup": 0, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": cb["sample_seconds"] * 1e3,
            "ms_per_step_c3_equivalent": 1e3 / cb["value"], "wall_s": wall,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded jittered grid + AS241 normals, simgen conventions)", "impl": "reference",
            "config": bench_config(args, cfgd["g"] ** 2, cfgd, 1),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "note": "reference is C++/Eigen and cannot be built here (Eigen absent); the arm times "
                    "oracle/ (CPU restatement, kind=port): ONE bounded sample (steps = 1 is what ran; "
                    "ms_per_step is the sample's own time), value = the C3-equivalent rate"}
    print(json.dumps(line), flush=True)


def _spawn_rank(rank, ws, port, argv):
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(ws),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    sys.argv = [sys.argv[0]] + argv
    main()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--c3-batch", action="store_true", help="also time a 9-θ batch at C3 (≈ 2 min)")
    ap.add_argument("--ref-g", type=int, default=256,
                    help="grid side of the reference arm's CPU sample (48, 96, 128, 192, 256 or 512)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # not under torchrun: spawn the N ranks here (one process per GPU, NCCL)
        import socket
        import torch.multiprocessing as mp
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        mp.spawn(_spawn_rank, args=(args.gpus, port, sys.argv[1:]), nprocs=args.gpus, join=True)
        return
    run_ours(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""HPS build+solve benchmark (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1]): 2D variable-coefficient Helmholtz
Delta u + k^2 (1 + q(x)) u = f on [-1,1]^2, DtN HPS, p = 16, uniform quadtree
L = 8 (65,536 leaves, N = 16,777,216 DOF), q = 10 seeded Gaussian bumps,
manufactured plane-wave solution (synthetic data, k = 30, away from box resonances).

One step = one full build (leaf stage + all merge levels) + one solve (downward
pass + leaf reconstruction) through the C-ABI (libhps_b200.so).  `value` is
DOF/s with the problem descriptor and the root boundary data resident on the
device; `e2e` is the same step through hpsg_solve with HOST buffers (boundary
data H2D, the whole solution field D2H inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference times the REFERENCE itself on the host cores: its own unmodified
sources (/root/reference/proj/src) compiled against an Eigen-API shim into
oracle/_ref/libhps_ref.so, serial loops as written + threaded BLAS on every core;
each step is a bounded sample scaled to the full L=8 step (bench.py reference_sample).

Under torchrun (N>1) the default is the north star's subtree-sharded run (strong scaling:
ONE L=8 problem over N GPUs, paper_2503_17535_b200/sharded.py): each rank builds its
subtrees, ships subtree-root [h|T] over NCCL to the owners of the few top merges, and the
boundary data comes back down; `value` = N_DOF / (max over ranks of the step time).
--mode replicas runs N independent full problems instead (weak scaling).
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
sys.path.insert(0, ROOT)

METRIC = "HPS build+solve seconds & DOF/s (2D p=16 L=8) at 1/2/4/8 B200; rel err vs oracle"
# PAPER.md:629 / :1755 -- H100 JAX, subtree recomputation, p=16 L=8: 4.02 s (N = 16,777,216)
PAPER_H100_DOFS = 16777216 / 4.02
FP64_PEAK_TFLOPS = 37.155     # DMMA microbench: profiles/r01_fp64_peak.json 37.155, re-measured with SM clocks at 1965 MHz in profiles/r02_fp64_peak.json 37.148 (MEASURED_PEAKS.json has no FP64 entry)
# dram__bytes_read.sum + dram__bytes_write.sum of one leaf-stage launch at p=16 L=8, per leaf kernel
# (ncu --set full of the current kernels, profiles/r02_ncu_summary.md)
LEAF_KERNEL_DRAM_BYTES = {"leaf_fused_kernel": 18.89e9 + 69.29e9, "leaf_fdm_kernel": 5.675e9 + 7.492e9}


def leaf_roofline(kernel, n_leaves, ref_flops, t_leaf_ms, exec_flops, traffic):
    """Roofline of the leaf-stage launch (the dominant single kernel of stage 1).  LU leaf kernels: achieved =
    SURVEY 8d F_leaf x leaves / the live launch time.  Fast-diagonalisation kernel: it executes fewer FLOPs than
    the reference's LU algorithm, so achieved = the FP64 tensor FLOPs it executed (DMMA.8x8x4 count x 512,
    counted on the device) / the launch time; the reference-algorithm rate is reported beside it."""
    r = {"bound": "tensor", "kernel": f"{kernel} (stage 1, all {n_leaves:,} leaves, one launch)", "peak": FP64_PEAK_TFLOPS,
         "unit": "TFLOP/s", "traffic": traffic, "launch_ms": t_leaf_ms,
         "peak_source": "FP64 DMMA microbench profiles/r01_fp64_peak.json (of measured)"}
    ref_rate = ref_flops / (t_leaf_ms / 1e3) / 1e12
    if exec_flops:
        rate = exec_flops / (t_leaf_ms / 1e3) / 1e12
        r.update({"achieved": rate, "frac": rate / FP64_PEAK_TFLOPS, "algorithmic_flops": exec_flops,
                  "flops_basis": "executed DMMA FLOPs of the fast-diagonalisation solve (device count)",
                  "reference_algorithm_flops": ref_flops, "reference_algorithm_equiv_tflops": ref_rate})
    else:
        r.update({"achieved": ref_rate, "frac": ref_rate / FP64_PEAK_TFLOPS, "algorithmic_flops": ref_flops,
                  "flops_basis": "SURVEY 8d F_leaf x leaves (the reference's LU local solve)"})
    return r


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.samples, self.proc, self.gpu = [], None, gpu_index

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "n_samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_b200(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_setup()
    local %= max(1, torch.cuda.device_count())   # gloo functional runs: several ranks per GPU
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "gloo":   # one-GPU functional check of the sharded path (host-staged P2P)
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if args.mode == "sharded":
            return run_sharded(args, world, rank, local)
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import problems as PR

    prob = PR.helmholtz_bumps(k=args.k, seed=args.seed)
    tree = H.build_uniform_tree(prob.lo, prob.hi, args.L, 2, args.p)
    N = tree.total_points
    solver = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=not args.explicit_root,
                         device=local)
    stream = torch.cuda.current_stream()
    solver.set_stream(stream.cuda_stream)

    g_host = prob.boundary(solver.root_boundary_points())
    g_dev = torch.tensor(g_host, device="cuda")
    u_dev = torch.empty((tree.n_leaves, tree.p ** 2), dtype=torch.float64, device="cuda")
    g_pin = torch.tensor(g_host).pin_memory()
    u_pin = torch.empty((tree.n_leaves, tree.p ** 2), dtype=torch.float64).pin_memory()

    def step_device():
        solver.build()
        solver.solve_device(g_dev.data_ptr(), 1, u_dev.data_ptr())

    def step_e2e():
        solver.build()
        H.lib().hpsg_solve(solver._h, H.hps._dp(g_pin.numpy()), 1, H.hps._dp(u_pin.numpy()), None)

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    st = solver.stats()
    launches_per_step = st["launches_build"] + st["launches_solve"]

    def timed(fn, K):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        builds, solves = [], []
        for _ in range(K):
            fn()
            s = solver.stats()
            builds.append(s["t_build_ms"])
            solves.append(s["t_solve_ms"])
            leaf_ms.append(s["t_leaf_ms"])
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms, float(np.mean(builds)), float(np.mean(solves))

    leaf_ms = []
    clocks = ClockSampler(local)
    clocks.start()
    ms, t_build, t_solve = timed(step_device, args.steps)
    t_leaf = float(np.mean(leaf_ms))
    clk = clocks.stop()
    u_gpu = u_dev.cpu().numpy()
    ms_e2e = ms
    if not args.profile:
        step_e2e()  # untimed warm-up of the host-buffer path (first call allocates its staging)
        torch.cuda.synchronize()
        ms_e2e, _, _ = timed(step_e2e, max(1, args.steps // 2))
    st = solver.stats()
    gemm_live = None
    if not args.profile:
        # one extra (untimed) build with every DMMA GEMM launch bracketed by CUDA events on its own
        # stream: the GEMM's summed launch time and its executed 2mnk FLOPs (block-sparse runs only)
        import ctypes as C
        lib = H.lib()
        lib.hpsg_dev_gemm_timing.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                             C.POINTER(C.c_longlong)]
        gms, gfl, gn = C.c_double(), C.c_double(), C.c_longlong()
        lib.hpsg_dev_gemm_timing(1, None, None, None)
        solver.build()
        rc = lib.hpsg_dev_gemm_timing(2, C.byref(gms), C.byref(gfl), C.byref(gn))
        lib.hpsg_dev_gemm_timing(0, None, None, None)
        if rc == 0 and gms.value > 0:
            gemm_live = {"ms": gms.value, "flops": gfl.value, "launches": gn.value}

    err_exact = PR.rel_linf(u_gpu, prob.exact(solver.leaf_points()))
    ni, ne, nb, npt = (args.p - 2) ** 2, 4 * args.p - 4, 4 * (args.p - 2), args.p ** 2
    leaf_flops = tree.n_leaves * (2 / 3 * ni ** 3 + 2 * ni * ni * ne + 2 * ni * ne * nb + 2 * nb * npt * nb
                                  + 2 * ni * ni + 2 * nb * npt)
    peaks = load_peaks()
    flops = st["build_flops"]
    leaf_kernel = {0: "leaf_fused_kernel", 2: "leaf_fdm_kernel", 3: "leaf_fdm_kernel"}.get(st["leaf_path"],
                                                                                           "batched leaf LU")
    value = N * world / (ms / 1e3)
    out = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / world / PAPER_H100_DOFS,
        "vs_baseline_ref": "per-GPU DOF/s / 4.17e6 DOF/s (PAPER.md:629, H100 JAX subtree recompute, p=16 L=8, 4.02 s)",
        "dtype": "f64", "data": "synthetic (seeded bump potential, manufactured plane wave; coefficients evaluated on device)",
        "config": workload_config(args, world),
        "parallelism": f"{world} independent replica(s)",
        "sign": "corrected (v=+L^-1 f); literal differs only in the sign of f",
        "stages_ms": {"build": t_build, "leaf": st["t_leaf_ms"], "merge": st["t_merge_ms"], "solve": t_solve,
                      "merge_by_depth": [round(x, 3) for x in st["t_level_ms"]]},
        # dominant single kernel: the leaf stage (one launch per build).  achieved = SURVEY 8d leaf FLOPs
        # (the reference algorithm's F_leaf) x leaves / the live CUDA-event time of that launch; the
        # fast-diagonalisation kernel also reports the FP64 tensor FLOPs it executed (device DMMA count);
        # traffic = dram read+write of that launch from the ncu --set full capture (profiles/)
        "roofline": leaf_roofline(leaf_kernel, tree.n_leaves, leaf_flops, t_leaf, st["leaf_exec_flops"],
                                  LEAF_KERNEL_DRAM_BYTES.get(leaf_kernel) if (args.L, args.p) == (8, 16) else None),
        "roofline_build": {"bound": "tensor", "kernel": "whole build (leaf kernel + batched DMMA LU/TRSM/GEMM merges)",
                           "achieved": flops / (t_build / 1e3) / 1e12, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                           "frac": flops / (t_build / 1e3) / 1e12 / FP64_PEAK_TFLOPS, "algorithmic_flops": flops,
                           "note": "SURVEY 8d dense-equivalent counts (a rate equivalent to the reference algorithm, not executed FLOPs): the block-sparse Schur products skip zero blocks and the rows of [h|T] on the domain boundary, which nothing reads (executed GEMM FLOPs: roofline_gemm)"},
        # the leaf kernel above is the one the round-1 review named; by launch-time share the dominant kernel is now
        # the DMMA GEMM (all launches together ~49 % of the step, profiles/r02_launch_summary_v3.txt), whose live
        # roofline is roofline_gemm (the largest launch keeps the DMMA pipe 91 % active, profiles/r02_gemm_d1_*)
        "dominant_kernel": "dgemm_tma_kernel (roofline_gemm)",
        "roofline_gemm": None if gemm_live is None else {
            "bound": "tensor", "kernel": f"dgemm_tma_kernel (all {gemm_live['launches']} build launches: LU trailing "
                                         "updates + block-sparse Schur products)",
            "achieved": gemm_live["flops"] / (gemm_live["ms"] / 1e3) / 1e12, "peak": FP64_PEAK_TFLOPS,
            "unit": "TFLOP/s", "frac": gemm_live["flops"] / (gemm_live["ms"] / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
            "algorithmic_flops": gemm_live["flops"], "launch_ms_sum": gemm_live["ms"],
            "note": "live CUDA events per launch on its stream, one extra untimed build; executed 2mnk FLOPs"},
        "solve_roofline": {"bound": "hbm", "achieved": st["solve_bytes"] / (t_solve / 1e3) / 1e9,
                           "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                           "frac": st["solve_bytes"] / (t_solve / 1e3) / 1e9 / peaks.get("hbm_gbs", 6532.5),
                           "algorithmic_bytes": st["solve_bytes"]},
        "e2e": {"value": N * world / (ms_e2e / 1e3), "unit": "DOF/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": int(g_host.nbytes), "d2h_bytes_per_step": int(u_pin.numpy().nbytes)},
        "gpu_launches": int(launches_per_step * args.steps),
        "accuracy": {"rel_linf_vs_exact": err_exact, "min_leaf_rcond": st["min_rcond"]},
        "clocks": clk,
        "device_gb": st["device_bytes"] / 1e9,
    }
    if world == 1 and not args.no_extras and not args.profile:
        out["configs_extra"] = {"config3_multi_rhs": bench_multi_rhs(solver, tree, torch, args)}
    del solver
    if world == 1 and not args.no_extras and not args.profile:
        out["configs_extra"]["config3_new_sources"] = bench_new_sources(torch, args)
        out["configs_extra"]["config4_3d"] = bench_3d(torch)
        out["configs_extra"]["iti_scatter2d"] = bench_iti(torch)
        out["configs_extra"]["subtree_recompute_L8"] = bench_recompute(torch, args, 8, 2)
        out["configs_extra"]["subtree_recompute_L9"] = bench_recompute(torch, args, 9, 2)
        out["configs_extra"]["planner_L9_80GB"] = bench_planner(args, 9, 80e9)
        out["configs_extra"]["config5_adaptive_3d"] = bench_adaptive(torch)
        out["configs_extra"]["cpp_adapter_e2e_L8"] = bench_adapter_e2e(torch, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = reference_sample(args, prob)
        out["cpu_baseline_parallel_port"], par = parallel_port_baseline(args, prob, u_gpu)
        out["accuracy"].update(par)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def bench_multi_rhs(solver, tree, torch, args, nrhs=256, chunk=64):
    """BASELINE configs[2]: 256 new boundary right-hand sides against the stored factorization
    (downward pass + leaf reconstruction as DMMA GEMMs, chunks of 64 RHS)."""
    gen = torch.Generator(device="cuda").manual_seed(args.seed)
    G = torch.randn((nrhs, solver.nb_root), dtype=torch.float64, device="cuda", generator=gen)
    U = torch.empty((chunk, tree.n_leaves, tree.p ** 2), dtype=torch.float64, device="cuda")
    solver.solve_device(G[:chunk].data_ptr(), chunk, U.data_ptr())   # warm-up (workspace)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for c0 in range(0, nrhs, chunk):
        solver.solve_device(G[c0:c0 + chunk].data_ptr(), chunk, U.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # linearity spot check: solve(2 g0 - g1) = 2 u0 - u1 on the last chunk
    g2 = (2 * G[nrhs - chunk] - G[nrhs - chunk + 1]).reshape(1, -1).contiguous()
    u2 = torch.empty((1, tree.n_leaves, tree.p ** 2), dtype=torch.float64, device="cuda")
    solver.solve_device(g2.data_ptr(), 1, u2.data_ptr())
    lin = float(((u2[0] - (2 * U[0] - U[1])).abs().max() / U[0].abs().max()).item())
    st = solver.stats()   # of the single-RHS solve above: stored operator bytes + one u
    flops_rhs = 2.0 * (st["solve_bytes"] - 8.0 * tree.total_points) / 8.0   # one FMA per stored operator entry
    return {"workload": f"2D Helmholtz p={tree.p} L={tree.L}: {nrhs} boundary RHS (seeded N(0,1)) on one build, "
                        f"chunks of {chunk}", "ms": ms, "ms_per_rhs": ms / nrhs,
            "rhs_dof_per_s": nrhs * tree.total_points / (ms / 1e3), "flops_per_rhs": flops_rhs,
            "achieved_tflops": flops_rhs * nrhs / (ms / 1e3) / 1e12, "linearity_rel": lin}


def bench_new_sources(torch, args, nsrc=256, chunk=32):
    """BASELINE configs[2] (ii): 256 new SOURCE right-hand sides against one stored build
    (HpsSolver::solve_new_source: leaf re-solves -- the fast-diagonalisation iteration on the new sources where
    the leaves allow it, else the kept LU factors -- the upward source pass through the stored merge factors,
    then the downward pass), chunks of 32 sources."""
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import problems as PR
    prob = PR.helmholtz_bumps(k=args.k, seed=args.seed)
    tree = H.build_uniform_tree(prob.lo, prob.hi, args.L, 2, args.p)
    s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=not args.explicit_root,
                    keep_factors=True)
    s.build()
    pts = torch.tensor(s.leaf_points(), device="cuda")
    g = torch.tensor(prob.boundary(s.root_boundary_points()), device="cuda")
    F = torch.empty((chunk, tree.n_leaves, tree.p ** 2), dtype=torch.float64, device="cuda")
    G = g.reshape(1, -1).repeat(chunk, 1).contiguous()
    U = torch.empty_like(F)
    for i in range(chunk):  # seeded smooth sources
        F[i] = torch.sin((1.0 + 0.1 * i) * pts[..., 0] - 0.5 * pts[..., 1] + 0.01 * i)
    s.solve_new_source_device(F.data_ptr(), G.data_ptr(), chunk, U.data_ptr())  # warm-up (workspace)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(nsrc // chunk):
        s.solve_new_source_device(F.data_ptr(), G.data_ptr(), chunk, U.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = s.stats()
    s.close()
    return {"workload": f"2D Helmholtz p={tree.p} L={tree.L}: {nsrc} source RHS (smooth seeded fields) + boundary "
                        f"data on one keep_factors build (leaf path {st['leaf_path']}: 2 = fast-diagonalisation re-solves, "
                        f"1 = kept LU factors), chunks of {chunk}",
            "ms": ms, "ms_per_source": ms / nsrc, "rhs_dof_per_s": nsrc * tree.total_points / (ms / 1e3),
            "build_ms_keep_factors": st["t_build_ms"], "device_gb": st["device_bytes"] / 1e9}


def bench_recompute(torch, args, L, depth, steps=1):
    """The paper's memory strategy (subtree recomputation, PAPER.md:629 -- the BASELINE.md number is
    this mode: 4.02 s at p=16 L=8 on an H100; L=9: 17.43 s): only the depth-`depth` subtree roots'
    [h|T] survive the build, each subtree is rebuilt for its downward pass (one reused workspace)."""
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import problems as PR
    from paper_2503_17535_b200.recompute import SubtreeRecomputeSolver
    prob = PR.helmholtz_bumps(k=args.k, seed=args.seed)
    tree = H.build_uniform_tree(prob.lo, prob.hi, L, 2, args.p)
    rs = SubtreeRecomputeSolver(tree, prob.terms, prob.source, depth=depth, literal_sign=False,
                                root_implicit_S=not args.explicit_root)
    g = torch.tensor(prob.boundary(rs.root_boundary_points()), device="cuda")
    u = torch.empty((1, tree.n_leaves, tree.p ** 2), dtype=torch.float64, device="cuda")
    rs.build()
    rs.solve_device(g, u)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        rs.build()
        rs.solve_device(g, u)
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / steps
    lib_bytes = rs.top.stats()["device_bytes"] + rs.work.stats()["device_bytes"]
    rs.close()
    paper = {8: 4.02, 9: 17.43}.get(L)
    return {"workload": f"2D Helmholtz p={tree.p} L={L} (N={tree.total_points}), subtree recomputation at depth "
                        f"{depth} (build + solve, wall clock)", "s_per_step": sec,
            "value": tree.total_points / sec, "unit": "DOF/s", "device_gb": lib_bytes / 1e9,
            "paper_h100_subtree_recompute_s": paper, "speedup_vs_paper": (paper / sec) if paper else None}


def bench_planner(args, L, budget):
    """SPEC planner make_plan on the real footprints (hpsg_estimate_bytes; nothing allocated): the
    store footprint of a 2D p=16 tree and the subtree plan under an H100-sized budget."""
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import planner as PL
    from paper_2503_17535_b200 import problems as PR
    prob = PR.helmholtz_bumps(k=args.k, seed=args.seed)
    tree = H.build_uniform_tree(prob.lo, prob.hi, L, 2, args.p)
    opts = dict(literal_sign=False, root_implicit_S=not args.explicit_root)
    whole = H.estimate_bytes(tree, prob.terms, prob.source, **opts)
    plan = PL.make_plan(tree, prob.terms, prob.source, strategy="subtree", budget=budget, **opts)
    return {"workload": f"planner: 2D Helmholtz p={tree.p} L={L} (N={tree.total_points}), budget {budget / 1e9:g} GB",
            "store_gb": whole / 1e9, "plan": plan.strategy, "cut_depth": plan.cut_depth,
            "subtree_height": plan.subtree_depth, "n_subtrees": plan.n_subtrees,
            "plan_peak_gb": plan.est_bytes.get("peak", plan.est_bytes.get("whole", 0.0)) / 1e9}


def bench_iti(torch, L=6, p=16, k=40.0, steps=2):
    """SURVEY 8f rank 1 (ItI variant): make_scattering (problems.cpp:109-152) with the radiation closure,
    build (leaf ItI maps, merge_iti, root T LU) + solve_radiation, complex128 in real-equivalent form."""
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import problems as PR
    pr = PR.scatter2d(k=k)
    tree = H.build_uniform_tree(-1.0, 1.0, L, 2, p)
    s = H.HpsSolver(tree, pr.terms, pr.source_re, source_imag=pr.source_im, variant="iti", eta=pr.eta,
                    build_root_T=True)
    s.build()
    s.solve_radiation()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        s.build()
        u = s.solve_radiation()
    ms = (time.perf_counter() - t0) / steps * 1e3
    st = s.stats()
    s.close()
    return {"workload": f"ItI scatter2d k={k:g}, p={p}, L={L} (N={tree.total_points}), radiation closure",
            "ms_per_step": ms, "value": tree.total_points / (ms / 1e3), "unit": "DOF/s (wall clock, host result)",
            "build_ms": st["t_build_ms"], "solve_ms": st["t_solve_ms"], "max_abs_u": float(np.abs(u).max())}


def bench_3d(torch, L=4, p=8, steps=2):
    """BASELINE configs[3]: 3D variable-coefficient Poisson div(eps grad u) = f, p=8, uniform
    octree L=4 (N = 2,097,152; root D = 27,648), one GPU (the 8-GPU octant sharding is the
    same sharded.py path with nchild = 8)."""
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import problems as PR
    prob = PR.poisson3d_var()
    tree = H.build_uniform_tree(prob.lo, prob.hi, L, 3, p)
    s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
    g = torch.tensor(prob.boundary(s.root_boundary_points()), device="cuda")
    u = torch.empty((tree.n_leaves, p ** 3), dtype=torch.float64, device="cuda")
    s.build()
    s.solve_device(g.data_ptr(), 1, u.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        s.build()
        s.solve_device(g.data_ptr(), 1, u.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    st = s.stats()
    err = PR.rel_linf(u.cpu().numpy(), prob.exact(s.leaf_points()))
    out = {"workload": f"3D variable-coefficient Poisson, p={p}, L={L} uniform octree, N={tree.total_points} DOF "
                       f"(BASELINE configs[3]), root D={st['top_D_size']} (implicit S)",
           "ms_per_step": ms, "value": tree.total_points / (ms / 1e3), "unit": "DOF/s",
           "build_ms": st["t_build_ms"], "solve_ms": st["t_solve_ms"],
           "merge_by_depth_ms": [round(x, 2) for x in st["t_level_ms"]],
           "counted_build_tflops": st["build_flops"] / st["t_build_ms"] / 1e9,
           "rel_linf_vs_exact": err, "device_gb": st["device_bytes"] / 1e9}
    s.close()
    return out


def bench_adapter_e2e(torch, args):
    """The headline workload through the reference-facing C++ drop-in (include/hps/hps_b200.hpp) as a caller
    of hps::HpsSolver<Real> writes it: std::function fields sampled on the host at all 16.8 M leaf points
    (every host core), build(), sample_root_data(), solve() into the per-leaf SolutionField
    (examples/adapter_e2e_b200.cpp, host clock).  The second of two runs is reported."""
    exe = os.path.join(ROOT, "examples", "adapter_e2e_b200")
    if not os.path.exists(exe):
        return {"skipped": "examples/adapter_e2e_b200 not built (make -C paper_2503_17535_b200 example)"}
    torch.cuda.empty_cache()
    r = subprocess.run([exe, str(args.L), "2", "0"], capture_output=True, text=True, timeout=900)
    if r.returncode != 0:
        return {"error": (r.stderr or r.stdout)[-400:]}
    rows = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    out = dict(rows[-1])
    out["note"] = ("host clock; t_setup = tree + host sampling of 3 std::function fields + upload; t_solve includes "
                   "sample_root_data, the H2D of g and the D2H of u into per-leaf vectors")
    return out


def bench_adaptive(torch):
    """SURVEY 8f rank 3 / BASELINE configs[4]: 3D adaptive octrees on the product's own mesher
    (refine_adaptive + enforce_level_restriction) and the general-tree pipeline (nonuniform merges).
    PAPER.md Table 1 (wavefront, p=8): uniform L=3 (top D 6912, 1.48e-4 in the paper) vs adaptive at matched
    error; config 5: Poisson-Boltzmann (smooth permittivity, 50 seeded centers), device memory logged."""
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import problems as PR
    from paper_2503_17535_b200.hps import FIELD_PB_EPS_GRAD, Field, GeneralTree, refine_adaptive

    def uniform(L, p, lo, hi):
        off = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
        depth, nch, ch, los, his = [0], [0], [[-1] * 8], [[lo] * 3], [[hi] * 3]
        for level in range(L):
            for i in [i for i, d in enumerate(depth) if d == level]:
                nch[i] = 8
                for c in range(8):
                    a, b = list(los[i]), list(his[i])
                    for k in range(3):
                        mid = 0.5 * (los[i][k] + his[i][k])
                        (a if off[c][k] else b)[k] = mid
                    ch[i][c] = len(depth)
                    depth.append(level + 1), nch.append(0), ch.append([-1] * 8), los.append(a), his.append(b)
        return GeneralTree(3, p, depth, nch, ch, los, his)

    def run(prob, tree, label, mesh_s=None):
        s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
        g = torch.tensor(prob.boundary(s.root_boundary_points()), device="cuda")
        u = torch.empty((tree.n_leaves, tree.p ** 3), dtype=torch.float64, device="cuda")
        s.build()
        s.solve_device(g.data_ptr(), 1, u.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.build()
        s.solve_device(g.data_ptr(), 1, u.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        st = s.stats()
        out = {"case": label, "n_leaves": tree.n_leaves, "N": tree.total_points, "top_D": st["top_D_size"],
               "max_leaf_depth": int(tree.depth[tree.leaves].max()), "ms_per_step": e0.elapsed_time(e1),
               "build_ms": st["t_build_ms"], "solve_ms": st["t_solve_ms"], "device_gb": st["device_bytes"] / 1e9}
        if mesh_s is not None:
            out["mesh_s_host"] = mesh_s
        if prob.exact is not None:
            out["rel_linf_vs_exact"] = PR.rel_linf(u.cpu().numpy(), prob.exact(s.leaf_points()))
        s.close()
        return out

    rows = []
    wf = PR.wavefront3d()
    rows.append(run(wf, uniform(3, 8, 0.0, 1.0), "wavefront3d uniform p=8 L=3"))
    for tol in (1e-2, 3e-5):
        t0 = time.perf_counter()
        tree, _ = refine_adaptive(0.0, 1.0, 8, [wf.source], tol=tol, max_depth=6)
        rows.append(run(wf, tree, f"wavefront3d adaptive p=8 tol={tol:g}", time.perf_counter() - t0))
    pb = PR.poisson_boltzmann3d()
    z, c = pb.source.centers, pb.terms[0].field.c
    fields = [Field(pb.source.kind, (0.0, 1.0, pb.source.c[2]), centers=z), pb.terms[0].field]
    fields += [Field(FIELD_PB_EPS_GRAD, tuple(c) + (float(a),), centers=z) for a in range(3)]
    t0 = time.perf_counter()
    tree, _ = refine_adaptive(-1.0, 1.0, 8, fields, tol=1e-2, max_depth=5)
    rows.append(run(pb, tree, "poisson_boltzmann3d adaptive p=8 tol=1e-2", time.perf_counter() - t0))
    return {"workload": "3D adaptive octrees (product mesher, nonuniform merges on the B200), corrected sign",
            "paper_table1_p8": {"uniform_D": 6912, "uniform_err": 1.48e-4, "adaptive_D": 2700, "adaptive_err": 1.45e-4},
            "runs": rows, "peak_device_gb": max(r["device_gb"] for r in rows)}


def run_sharded(args, world, rank, local):
    """Subtree-sharded strong-scaling step on N GPUs of one node."""
    import torch
    import torch.distributed as dist
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import problems as PR
    from paper_2503_17535_b200 import sharded as SH

    dist.barrier()   # communicators up on every rank before the first (partial) point-to-point batch
    prob = PR.helmholtz_bumps(k=args.k, seed=args.seed)
    tree = H.build_uniform_tree(prob.lo, prob.hi, args.L, 2, args.p)
    N = tree.total_points
    plan = SH.make_plan(args.L, 2, world)
    parts = SH.CudaParts(tree, prob.terms, prob.source, literal_sign=False,
                         root_implicit_S=not args.explicit_root, device=local)
    shard = SH.ShardedHps(plan, rank, parts)
    stream = torch.cuda.current_stream()
    g_host = prob.boundary(H.tree_root_points(tree)) if rank == 0 else None
    g_dev = torch.tensor(g_host, device="cuda").reshape(1, -1) if rank == 0 else None
    g_pin = torch.tensor(g_host).reshape(1, -1).pin_memory() if rank == 0 else None
    all_parts = list(shard.sub.values()) + list(shard.top.values())
    on_dev = dist.get_backend() == "nccl"

    def reduce(vals, op):
        t = torch.tensor(vals, dtype=torch.float64, device="cuda" if on_dev else "cpu")
        dist.all_reduce(t, op=op)
        return t.tolist()

    def step_device():
        return SH.run_dist(shard, g_dev, nrhs=1)

    def step_e2e():
        g = g_pin.to("cuda", non_blocking=True) if rank == 0 else None
        u = SH.run_dist(shard, g, nrhs=1)
        return {k: v.to("cpu") for k, v in u.items()}

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    def timed(fn, K):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(K):
            out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return reduce([e0.elapsed_time(e1) / K], dist.ReduceOp.MAX)[0], out

    clocks = ClockSampler(local)
    clocks.start()
    ms, u = timed(step_device, args.steps)
    clk = clocks.stop()
    ms_e2e = ms
    if not args.profile:
        step_e2e()  # untimed warm-up of the host-buffer path
        torch.cuda.synchronize()
        ms_e2e, _ = timed(step_e2e, max(1, args.steps // 2))
    # job-wide counters: counted FLOPs, launches, leaf/merge times of this rank's parts
    loc = reduce([sum(p.stats()["build_flops"] for p in all_parts),
                  sum(p.stats()["launches_build"] + p.stats()["launches_solve"] for p in all_parts),
                  sum(p.stats()["t_build_ms"] for p in all_parts)], dist.ReduceOp.SUM)
    # accuracy on this rank's leaves against the manufactured solution
    err = 0.0
    for k, part in shard.sub.items():
        ex = prob.exact(part.s.leaf_points())
        err = max(err, float(np.abs(u[k][0].cpu().numpy() - ex).max() / np.abs(ex).max()))
    err = reduce([err], dist.ReduceOp.MAX)[0]
    flops, launches = loc[0], int(loc[1])
    value = N / (ms / 1e3)
    up = 0
    for d in range(plan.ds):
        for i in range(plan.nchild ** d):
            for c in range(plan.nchild):
                if plan.owner(d + 1, plan.nchild * i + c) != plan.owner(d, i):
                    nb = 4 * tree.q * 2 ** (args.L - 1 - d)   # boundary points of a depth-(d+1) node
                    up += 8 * (1 + nb) * nb
    out = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": value / PAPER_H100_DOFS,
        "vs_baseline_ref": "job DOF/s / 4.17e6 DOF/s (PAPER.md:629, 1x H100 JAX subtree recompute, p=16 L=8, 4.02 s)",
        "dtype": "f64", "data": "synthetic (seeded bump potential, manufactured plane wave; coefficients evaluated on device)",
        "config": workload_config(args, world),
        "parallelism": f"subtree-sharded over {world} GPUs: cut depth {plan.ds}, "
                       f"{plan.n_sub} subtrees, NCCL P2P of {up / 1e6:.0f} MB [h|T] up per build",
        "sign": "corrected (v=+L^-1 f); literal differs only in the sign of f",
        "roofline": {"bound": "tensor", "kernel": "build (batched DMMA LU/TRSM/GEMM pipeline), whole job",
                     "achieved": flops / (ms / 1e3) / 1e12, "peak": FP64_PEAK_TFLOPS * world, "unit": "TFLOP/s",
                     "frac": flops / (ms / 1e3) / 1e12 / (FP64_PEAK_TFLOPS * world), "traffic": None,
                     "algorithmic_flops": flops, "note": "counted build FLOPs over the whole build+solve step time"},
        "e2e": {"value": N / (ms_e2e / 1e3), "unit": "DOF/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": int(8 * tree.root_boundary_size),
                "d2h_bytes_per_step": int(8 * N)},
        "gpu_launches": launches * args.steps,
        "accuracy": {"rel_linf_vs_exact": err},
        "clocks": clk,
    }
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def workload_config(args, world):
    """The `config` object of both arms (identical dicts, so the driver can pair them)."""
    N = (4 ** args.L) * args.p ** 2
    return {"workload": f"2D variable-coefficient Helmholtz DtN HPS, p={args.p}, L={args.L} uniform quadtree, "
                        f"N={N} DOF (BASELINE configs[1])", "k": args.k, "seed": args.seed,
            "root": "explicit S" if args.explicit_root else "implicit S (MergeOptions::implicit_S)",
            "l2": "inputs larger than L2 (each step streams > 40 GB of leaf/merge operands)"}


def _oracle_terms(prob):
    from oracle import oracle as O
    keep, terms = [], []
    for t in prob.terms:
        f, k = O.make_field(t.field.kind, t.field.c, t.field.centers, t.field.samples)
        keep += k
        terms.append((t.role, t.axis, t.axis2, f))
    src, k = O.make_field(prob.source.kind, prob.source.c, prob.source.centers, prob.source.samples)
    keep += k
    return terms, src, keep


def reference_sample(args, prob, m=None):
    """The REFERENCE's own build + solve (oracle/_ref: /root/reference/proj/src unmodified + the Eigen-API
    shim) on the host cores, as written: serial leaf and merge loops, BLAS (Eigen's OpenMP GEMM in the
    original build) on every core.  A full L=8 step takes minutes, so each step is a bounded sample scaled
    to the whole step (ref_capi.h ref_bench_sample): one depth-(L-m) subtree built and solved end to end by
    the reference x 4^(L-m), plus one reference merge_node + propagate step per top depth x 4^d."""
    from oracle import ref as R
    threads = os.cpu_count()
    R.set_threads(threads)
    m = m if m is not None else min(args.L, 5)
    terms, src, keep = _oracle_terms(prob)
    est = R.bench_sample(args.p, args.L, m, prob.lo, prob.hi, terms, src, root_implicit=not args.explicit_root)
    N = (4 ** args.L) * args.p ** 2
    top = args.L - m
    sample = (f"reference HpsSolver build+solve of one depth-{top} subtree ({est['sub_leaves']} leaves, "
              f"{est['sub_build_s']:.2f} s + {est['sub_solve_s']:.3f} s) x {4 ** top}, plus one reference "
              f"merge_node + propagate per depth d < {top} (" +
              ", ".join(f"d{d}: {est['merge_s'][d]:.2f}+{est['propagate_s'][d]:.3f} s x {4 ** d}" for d in range(top)) +
              f"); estimated full step {est['est_s']:.1f} s")
    return {"value": N / est["est_s"], "unit": "DOF/s", "cores": threads, "kind": "reference",
            "schedule": "reference-faithful: serial leaf/merge loops (solver.cpp:144-151), threaded BLAS",
            "sample": sample, "est_step_s": est["est_s"]}


def parallel_port_baseline(args, prob, u_gpu=None):
    """The oracle restatement (C++ port) on the host cores with OpenMP over leaves and merges: the FULL
    workload, one build + solve (labelled: a parallel schedule the reference does not have)."""
    from oracle import oracle as O
    from tests.oracle_problems import oracle_solver
    threads = os.cpu_count()
    O.set_threads(threads)
    s = oracle_solver(prob, args.p, args.cpu_L, literal=False, root_implicit=not args.explicit_root, parallel=True)
    t0 = time.perf_counter()
    s.build()
    t1 = time.perf_counter()
    g = prob.boundary(s.root_points())
    u = s.solve(g)
    t2 = time.perf_counter()
    N = s.n_leaves * s.npts
    res = {"value": N / (t2 - t0), "unit": "DOF/s", "cores": threads, "kind": "port",
           "schedule": "parallel port: OpenMP over leaves and over the merges of a level + threaded OpenBLAS",
           "sample": f"full workload at L={args.cpu_L} (N={N}), one build+solve; build {t1 - t0:.2f} s, "
                     f"solve {t2 - t1:.2f} s"}
    par = {}
    if u_gpu is not None and args.cpu_L == args.L:
        par["rel_linf_vs_oracle"] = float(np.abs(u_gpu - u).max() / np.abs(u).max())
        par["parity_tol"] = 1e-10
        par["parity_ok"] = bool(par["rel_linf_vs_oracle"] <= 1e-10)
    return res, par


def native_libs():
    """Shared objects of this repo mapped into the process (the reference arm must map only oracle/)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {line.split()[-1] for line in f if line.rstrip().endswith(".so") and ROOT in line}
        return sorted(os.path.relpath(p, ROOT) for p in paths)
    except OSError:
        return []


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    from paper_2503_17535_b200 import problems as PR   # descriptors only: no shared object is loaded
    prob = PR.helmholtz_bumps(k=args.k, seed=args.seed)
    vals, res = [], None
    for i in range(args.warmup + args.steps):
        res = reference_sample(args, prob)
        if i >= args.warmup:
            vals.append(res["value"])
    value = float(np.median(vals))
    libs = native_libs()
    if any("libhps_b200" in x for x in libs):
        raise SystemExit("reference arm mapped the product library: " + ", ".join(libs))
    out = {"metric": METRIC, "impl": "reference", "value": value, "unit": "DOF/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": (4 ** args.L) * args.p ** 2 / value * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded bump potential, manufactured plane wave)",
           "config": workload_config(args, world),
           "cpu_baseline": dict(res, value=value),
           "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "native_libs": libs}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: host-staged transport, for functional runs of N ranks on one GPU")
    ap.add_argument("--mode", choices=["sharded", "replicas"], default="sharded",
                    help="N>1: subtree-sharded strong scaling (default) or independent replicas")
    ap.add_argument("--L", type=int, default=8)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--k", type=float, default=30.0)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--cpu-L", type=int, default=None, help="tree depth of the CPU baseline run (default: --L)")
    ap.add_argument("--explicit-root", action="store_true", help="form S at the root (reference 2D default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the config 3 (256 RHS) and config 4 (3D) lines")
    ap.add_argument("--profile", action="store_true", help="one untimed-warmup-free step for ncu launch lists")
    args = ap.parse_args()
    if args.profile:
        args.steps, args.warmup, args.no_cpu_baseline = 1, 0, True
    if args.cpu_L is None:
        args.cpu_L = args.L
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

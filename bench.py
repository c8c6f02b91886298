"""Benchmark: MG-PCG solve of the SIMP elasticity system on one B200 per rank.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl b200|reference]

A step is one drop-in call of the hot path on the config's workload, for every
solver leg the config names (config 1: GMG 5 levels AND SA-AMG on identical
inputs): element moduli from rho, K(rho), hierarchy build, PCG to rtol=1e-8,
compliance and sensitivity -- what one topology-optimisation iteration costs
(the reference rebuilds the preconditioner every iteration).
Metric: DOF*iterations/s (higher is better) = sum(ndof*iters) / sum(step time).
Inputs are resident in HBM when the timed region starts; L2 is flushed before
every timed step.  ``e2e`` repeats the metric through the C-ABI host-buffer entry
point (tmg_solve_compliance_host) with H2D/D2H copies inside the timed region.
``--impl reference`` times the CPU oracle port of the reference algorithm on a
bounded sample (setup + a fixed number of PCG iterations per leg) on rank 0.
Under torchrun every rank runs an independent replica (scaling: weak).
"""

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MG-PCG DOF*iterations/s (setup+solve+sensitivity per step)"
UNIT = "DOF*iter/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--cpu-sample-iters", type=int, default=10)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--iters-cap", type=int, default=0,
                   help="profiling only: cap every leg's PCG iterations (ncu launch lists)")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def replica_throughput(local_ms, local_work, world, device):
    """Whole-job throughput of N independent replicas: every rank did the same
    work; the job took as long as the slowest rank (max over ranks of the
    device-timed region).  Returns (max_ms, units/s)."""
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.barrier()
        t = torch.tensor([local_ms], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        local_ms = float(t.item())
    return local_ms, world * local_work / (local_ms / 1e3)


def config_dict(w, args, world):
    from paper_2001_01655_b200 import problems
    return {"workload": w.name, "config_index": args.config, "ndof": int(w.ndof),
            "elements": int(w.mesh.element_count), "legs": [problems.leg_name(s) for s in w.solvers],
            "rtol": w.rtol, "precision": "fp64", "l2": "flushed (256 MiB write) before every timed step",
            "parallelism": "replicas x%d" % world}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.err = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable: %s" % self.err]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def oracle_sample(w, leg, iters, threads=1):
    """threads=1: the scalar cpu_baseline of the B200 line; the --impl reference arm
    passes every host thread (numpy BLAS may use them; scipy's sparse kernels are
    single-threaded)."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(threads):
        return _oracle_sample(w, leg, iters)


def _oracle_sample(w, leg, iters):
    from oracle import topomg_oracle as O
    from paper_2001_01655_b200 import problems
    g = O.make_grid(w.mesh.dims)
    t0 = time.perf_counter()
    E = O.simp_modulus(w.rho, problems.PENAL, problems.E0, problems.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    if leg["smoother"] == "chebyshev":
        sm = O.Smoother("chebyshev", 1.0, leg.get("degree", 2))
    else:
        sm = O.Smoother(leg["smoother"], leg.get("weight", 0.5), safeguard=leg.get("safeguard", 0.0))
    if leg["strategy"] == "gmg":
        h = O.build_gmg(g, K, 1, sm, leg["n_pre"], leg["n_post"], max_levels=leg["levels"])
    elif leg["strategy"] == "amg":
        h = O.build_sa_amg(K, O.rigid_body_modes(g, w.bc.fixed_dofs), leg["coarse_max_dofs"], sm, leg["n_pre"],
                           leg["n_post"], beta=leg["beta"], isolated=leg.get("isolated", "merge"))
    else:
        h = O.build_hybrid(g, K, O.rigid_body_modes(g, w.bc.fixed_dofs), leg["n_geo"], leg["coarse_max_dofs"], sm,
                           leg["n_pre"], leg["n_post"], beta=leg["beta"], isolated=leg.get("isolated", "merge"))
    u, rec = O.pcg(K, w.bc.load_vector, None, h.apply, rtol=w.rtol, max_iterations=iters)
    O.compliance_sensitivity(g, w.bc.load_vector, u, w.rho, problems.PENAL, problems.E0, problems.EMIN)
    dt = time.perf_counter() - t0
    return w.ndof * rec.iterations, dt, rec.iterations


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2001_01655_b200 import problems
    w = problems.CONFIGS[args.config]()
    work = secs = 0.0
    cores = os.cpu_count() or 1
    for step in range(args.warmup + args.steps):
        wk = dt = 0.0
        for leg in w.solvers:
            a, b, _ = oracle_sample(w, leg, args.cpu_sample_iters, threads=cores)
            wk += a
            dt += b
        if step >= args.warmup:
            work += wk
            secs += dt
    value = work / secs
    sample = ("oracle port (numpy/scipy, %d host threads allowed; its sparse kernels run on one): setup + %d PCG "
              "iterations per leg (%s) per step" % (cores, args.cpu_sample_iters,
                                                   ",".join(problems.leg_name(l) for l in w.solvers)))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json config %d)" % args.config,
            "config": config_dict(w, args, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
class LegRunner:
    """Device-resident inputs and the drop-in call sequence of one solver leg."""

    def __init__(self, w, leg):
        import torch

        import paper_2001_01655_b200 as T
        from paper_2001_01655_b200 import problems
        self.T, self.w, self.leg = T, w, leg
        self.name = problems.leg_name(leg)
        self.sm = problems.smoother_settings(leg)
        self.maxit = leg.get("max_iterations", 10000)
        self.isolated = leg.get("isolated", "merge")
        if leg["strategy"] == "amg":
            B = T.rigid_body_modes(w.mesh, w.bc.fixed_dofs)
            self.B = torch.as_tensor(B, device="cuda")
            self.v0 = torch.as_tensor(np.random.default_rng(0).standard_normal(w.ndof), device="cuda")
        elif leg["strategy"] == "hybrid":
            self.B = T.rigid_body_modes(w.mesh, w.bc.fixed_dofs)

    def build(self, K):
        T, w, leg = self.T, self.w, self.leg
        if leg["strategy"] == "gmg":
            return T.build_gmg(w.mesh, K, 1, self.sm, leg["n_pre"], leg["n_post"], max_levels=leg["levels"])
        if leg["strategy"] == "amg":
            return T.build_sa_amg(K, self.B, leg["coarse_max_dofs"], self.sm, leg["n_pre"], leg["n_post"],
                                  beta=leg["beta"], v0=self.v0, isolated=self.isolated)
        return T.build_hybrid(w.mesh, K, self.B, leg["n_geo"], leg["coarse_max_dofs"], self.sm, leg["n_pre"],
                              leg["n_post"], beta=leg["beta"], isolated=self.isolated)

    def mg_desc(self):
        """tmg_mg_desc for the host-buffer entry point (+ keep-alive host arrays)."""
        from paper_2001_01655_b200 import _lib
        from paper_2001_01655_b200.mesh import StructuredMesh, rigid_body_modes
        from paper_2001_01655_b200.multigrid import hybrid_plan
        from paper_2001_01655_b200.multigrid import isolated_mode as T_isolated_mode
        leg, w = self.leg, self.w
        mg = _lib.MgDesc()
        mg.strategy = {"gmg": 0, "amg": 1, "hybrid": 2}[leg["strategy"]]
        mg.coarse_max_dofs = leg.get("coarse_max_dofs", 1)
        mg.max_levels = leg.get("levels", 0)
        mg.smoother = self.sm.desc()
        mg.n_pre, mg.n_post = leg["n_pre"], leg["n_post"]
        keep = []
        if leg["strategy"] == "amg":
            B = np.ascontiguousarray(rigid_body_modes(w.mesh, w.bc.fixed_dofs))
            v0 = np.random.default_rng(0).standard_normal(w.ndof)
            keep = [B, v0]
        elif leg["strategy"] == "hybrid":
            dims, sizes, _ = hybrid_plan(w.mesh, leg["n_geo"], leg["coarse_max_dofs"])
            B = np.ascontiguousarray(rigid_body_modes(StructuredMesh(dims, sizes)))
            v0 = np.random.default_rng(0).standard_normal(B.shape[0])
            keep = [B, v0]
            mg.n_geo = leg["n_geo"]
        if keep:
            mg.beta = leg["beta"]
            mg.near_nullspace_host = keep[0].ctypes.data
            mg.nvec = keep[0].shape[1]
            mg.coarse_ndof = keep[0].shape[0]
            mg.v0_host = keep[1].ctypes.data
            mg.isolated_mode = T_isolated_mode(self.isolated)
        return mg, keep


def run_b200(args, rank, world, local):
    import torch

    import paper_2001_01655_b200 as T
    from paper_2001_01655_b200 import _lib, problems
    from paper_2001_01655_b200._dev import as_dev, empty_dev, ptr, stream_ptr

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = problems.CONFIGS[args.config]()
    runners = [LegRunner(w, leg) for leg in w.solvers]
    if args.iters_cap > 0:
        for lr in runners:
            lr.maxit = min(lr.maxit, args.iters_cap)
    L = _lib.load()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    rho_d = as_dev(w.rho)
    f_d = as_dev(w.bc.load_vector)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    state = {}

    def step():
        work = 0
        state["legs"] = []
        for lr in runners:
            E = law.modulus(rho_d)
            K = T.StiffnessOperator(w.mesh, w.bc, E)
            h = lr.build(K)
            u, rec = T.cg_solve(K, f_d, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=lr.maxit))
            dc = empty_dev(w.mesh.element_count)
            comp = C.c_double()
            _lib.check(L.tmg_compliance_sensitivity(K.handle, ptr(rho_d), ptr(f_d), ptr(u), law.penalty,
                                                    law.e_max, law.e_min, ptr(dc), C.byref(comp),
                                                    stream_ptr(None)))
            work += w.ndof * rec.iterations
            hist = rec.residual_history
            state["legs"].append({"leg": lr.name, "iterations": rec.iterations, "converged": rec.converged,
                                  "rel_residual": hist[-1] / hist[0], "solve_ms": rec.solve_time * 1e3,
                                  "max_iterations": lr.maxit, "compliance": comp.value,
                                  "levels": [lv.size for lv in h.levels]})
            state.setdefault("h", h)
        return work

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches0 = L.tmg_launch_count()
    total_ms, total_work = 0.0, 0
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            wk = step()
            e1.record()
            torch.cuda.synchronize()
            total_ms += e0.elapsed_time(e1)
            total_work += wk
    launches = L.tmg_launch_count() - launches0
    total_ms, value = replica_throughput(total_ms, total_work, world, "cuda")
    roof = roofline(args, w, state, L)
    e2e = e2e_run(args, w, runners, L, law, world)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json config %d)" % args.config,
            "config": config_dict(w, args, world), "leg_results": state["legs"],
            "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        wk = dt = 0.0
        for leg in w.solvers:
            a, b, _ = oracle_sample(w, leg, args.cpu_sample_iters)
            wk += a
            dt += b
        line["cpu_baseline"] = {"value": wk / dt, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": "oracle port (numpy/scipy, 1 thread): setup + %d PCG iterations of "
                                          "each leg, %.1f s" % (args.cpu_sample_iters, dt)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def roofline(args, w, state, L):
    import torch
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    h = state["h"]
    ms = C.c_double()
    from paper_2001_01655_b200._lib import check
    check(L.tmg_hierarchy_time_smoother(h.handle, 0, 50, C.byref(ms), torch.cuda.current_stream().cuda_stream))
    mesh = w.mesh
    d = mesh.ndim
    nodes, nel = mesh.node_count, mesh.element_count
    bytes_launch = nodes * (4 * 8 * d + 1) + nel * 8
    achieved = bytes_launch / (ms.value / 1e3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get("config%d" % args.config, {}).get("jacobi_dram_bytes")
    except Exception:  # noqa: BLE001
        pass
    return {"kernel": "k_jacobi<%d,FineOp> (level-0 weighted-Jacobi sweep, matrix-free K)" % d,
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "bytes_per_launch": bytes_launch, "launch_us": ms.value * 1e3,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
            "timing": "CUDA events around one replay of a CUDA graph of 50 back-to-back launches",
            "note": "working set %.1f MB vs 126 MB L2" % (bytes_launch / 1e6)}


def e2e_run(args, w, runners, L, law, world=1):
    from paper_2001_01655_b200 import _lib
    rho = np.ascontiguousarray(w.rho, dtype=np.float64)
    f = np.ascontiguousarray(w.bc.load_vector)
    fixed = np.ascontiguousarray(w.bc.fixed_dofs, dtype=np.int64)
    u = np.empty(w.ndof)
    dc = np.empty(w.mesh.element_count)
    comp = C.c_double()
    rec = _lib.SolveRec()
    md = _lib.mesh_desc(w.mesh)
    descs = [lr.mg_desc() for lr in runners]
    cfgs = [_lib.SolveDesc(w.rtol, lr.maxit) for lr in runners]

    def call():
        work = 0
        for (mg, keep), cfg in zip(descs, cfgs):
            _lib.check(L.tmg_solve_compliance_host(C.byref(md), rho.ctypes.data, fixed.ctypes.data, fixed.size,
                                                   f.ctypes.data, law.penalty, law.e_max, law.e_min, 0.3,
                                                   C.byref(mg), C.byref(cfg), u.ctypes.data, dc.ctypes.data,
                                                   C.byref(comp), C.byref(rec)))
            work += w.ndof * rec.iterations
        return work
    call()
    work = secs = 0.0
    for _ in range(max(1, args.e2e_steps)):
        t0 = time.perf_counter()
        work += call()
        secs += time.perf_counter() - t0
    h2d = sum(rho.nbytes + f.nbytes + w.mesh.node_count + 8 * 24 * 24 +
              sum(a.nbytes for a in keep) for (mg, keep) in descs)
    d2h = len(descs) * (u.nbytes + dc.nbytes + 16)
    # whole job over the replicas, timed as the slowest rank (as `value`)
    ms, value = replica_throughput(1e3 * secs, work, world, "cuda")
    secs = ms / 1e3
    return {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": 1e3 * secs / max(1, args.e2e_steps),
            "timing": "host wall clock around tmg_solve_compliance_host per leg (host buffers in/out)"}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()

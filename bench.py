"""Benchmark: MG-PCG solve of the SIMP elasticity system on one B200 per rank.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--iters 2] [--impl b200|reference]

Workload: BASELINE.json configs[4] (3D cantilever 192x96x96 Hex8, 5,455,809
nominal / 5,447,811 actual dofs, hybrid preconditioner: 3 geometric levels +
SA-AMG, Jacobi-Chebyshev), the largest single-GPU configuration (BASELINE.json
quotes its metric on no particular config).  Both arms build the operator and
the hierarchy ONCE per process (reported as ``setup_ms``, as the reference
reports setup and solve separately, optimization.py:372-387) and then time
identical steps: one PCG solve of exactly ``--iters`` iterations from x0 = 0
(none of the configs meets rtol 1e-8 on the true residual in fp64,
profiles/r02_attainable_accuracy.txt, so every solve runs to its cap) plus the
compliance f.u and the per-element sensitivity dc.
Metric: DOF*iterations/s (higher is better) = ndof * iterations / step time.
Inputs are resident in HBM when the timed region starts (working set > 0.9 GB,
far above the 126 MB L2; L2 is also flushed before every timed step).
``e2e`` repeats the step through the public Python API with HOST buffers: the
load vector copied from pinned host memory, u and dc read back, inside the
timed region.  ``--impl reference`` runs the CPU oracle port of the reference
algorithm (numpy/scipy) on the same config with the same --iters on rank 0.
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

METRIC = "MG-PCG DOF*iterations/s (fixed-iteration PCG solve + compliance sensitivity per step, setup once)"
UNIT = "DOF*iter/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=4)
    p.add_argument("--iters", type=int, default=2, help="PCG iterations per solve (both arms)")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--roofline-reps", type=int, default=20)
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
            "pcg_iterations_per_solve": args.iters, "rtol": w.rtol, "precision": "fp64",
            "step": "per leg: PCG solve of exactly %d iterations (x0 = 0) + compliance + sensitivity; operator and "
                    "hierarchy built once (setup_ms)" % args.iters,
            "l2": "working set > 0.9 GB (> 126 MB L2); also flushed (256 MiB write) before every timed step",
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
# CPU oracle (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
class OracleLegs:
    """The oracle port of the reference path on the host: operator + hierarchy
    built once (timed as setup), then steps of a fixed-iteration PCG solve plus
    compliance and sensitivity -- the same work per step as the B200 arm."""

    def __init__(self, w, threads=1):
        from oracle import topomg_oracle as O
        from paper_2001_01655_b200 import problems
        from threadpoolctl import threadpool_limits
        self.O, self.P, self.w, self.threads = O, problems, w, threads
        self.g = O.make_grid(w.mesh.dims)
        with threadpool_limits(threads):
            t0 = time.perf_counter()
            E = O.simp_modulus(w.rho, problems.PENAL, problems.E0, problems.EMIN)
            self.K = O.assemble_stiffness(self.g, w.bc.fixed_dofs, E)
            self.h = [self._build(leg) for leg in w.solvers]
            self.setup_s = time.perf_counter() - t0

    def _build(self, leg):
        O, w, g, K = self.O, self.w, self.g, self.K
        if leg["smoother"] == "chebyshev":
            sm = O.Smoother("chebyshev", 1.0, leg.get("degree", 2), lanczos_steps=leg.get("lanczos_steps", 10))
        else:
            sm = O.Smoother(leg["smoother"], leg.get("weight", 0.5), safeguard=leg.get("safeguard", 0.0))
        if leg["strategy"] == "gmg":
            return O.build_gmg(g, K, 1, sm, leg["n_pre"], leg["n_post"], max_levels=leg["levels"])
        if leg["strategy"] == "amg":
            return O.build_sa_amg(K, O.rigid_body_modes(g, w.bc.fixed_dofs), leg["coarse_max_dofs"], sm,
                                  leg["n_pre"], leg["n_post"], beta=leg["beta"], isolated=leg.get("isolated", "merge"))
        return O.build_hybrid(g, K, O.rigid_body_modes(g, w.bc.fixed_dofs), leg["n_geo"], leg["coarse_max_dofs"], sm,
                              leg["n_pre"], leg["n_post"], beta=leg["beta"], isolated=leg.get("isolated", "merge"))

    def step(self, iters):
        """(dof*iterations, seconds) of one step over every leg."""
        from threadpoolctl import threadpool_limits
        O, P, w = self.O, self.P, self.w
        work = 0
        with threadpool_limits(self.threads):
            t0 = time.perf_counter()
            for h in self.h:
                u, rec = O.pcg(self.K, w.bc.load_vector, None, h.apply, rtol=w.rtol, max_iterations=iters)
                O.compliance_sensitivity(self.g, w.bc.load_vector, u, w.rho, P.PENAL, P.E0, P.EMIN)
                work += w.ndof * rec.iterations
            return work, time.perf_counter() - t0


REF_WARMUP_CAP = 1  # CPU arm: one warm-up step (no caches/clocks to settle; a step costs ~10 s on config 4)


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2001_01655_b200 import problems
    w = problems.CONFIGS[args.config]()
    cores = os.cpu_count() or 1
    ol = OracleLegs(w, threads=cores)
    for _ in range(min(args.warmup, REF_WARMUP_CAP)):
        ol.step(args.iters)
    work = secs = 0.0
    for _ in range(args.steps):
        a, b = ol.step(args.iters)
        work += a
        secs += b
    value = work / secs
    sample = ("oracle port of the reference path (numpy/scipy; %d host threads allowed, scipy's sparse kernels run "
              "on one): operator + hierarchy once (%.1f s), then per step and leg (%s) a %d-iteration PCG solve + "
              "compliance + sensitivity on the full config-%d workload; %d warm-up step(s)" % (
                  cores, ol.setup_s, ",".join(problems.leg_name(l) for l in w.solvers), args.iters, args.config,
                  min(args.warmup, REF_WARMUP_CAP)))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "setup_ms": 1e3 * ol.setup_s, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, BASELINE.json config %d)" % args.config,
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
    L = _lib.load()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    rho_d = as_dev(w.rho)
    f_d = as_dev(w.bc.load_vector)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    cfg = T.SolveConfig(method="cg", rtol=w.rtol, max_iterations=args.iters)
    # setup once (timed): moduli, matrix-free operator, hierarchies
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    K = T.StiffnessOperator(w.mesh, w.bc, law.modulus(rho_d))
    hs = [lr.build(K) for lr in runners]
    s1.record()
    torch.cuda.synchronize()
    setup_ms = s0.elapsed_time(s1)
    dc = empty_dev(w.mesh.element_count)
    state = {"h": hs[0]}

    fnorm = float(np.linalg.norm(w.bc.load_vector))
    level_sizes = [[lv.size for lv in h.levels] for h in hs]

    def step():
        """One step: per leg the solve and the fused compliance + sensitivity; nothing
        else on the host between the device calls (the event-timed region would
        see it as GPU idle time)."""
        work, out = 0, []
        for h in hs:
            u, rec = T.cg_solve(K, f_d, None, h, cfg)
            comp = C.c_double()
            _lib.check(L.tmg_compliance_sensitivity(K.handle, ptr(rho_d), ptr(f_d), ptr(u), law.penalty,
                                                    law.e_max, law.e_min, ptr(dc), C.byref(comp),
                                                    stream_ptr(None)))
            work += w.ndof * rec.iterations
            out.append((rec, comp.value))
        state["last"] = out
        return work

    def leg_results():
        return [{"leg": lr.name, "iterations": rec.iterations, "converged": rec.converged,
                 "true_rel_residual": rec.residual_history[-1] / fnorm, "solve_ms": rec.solve_time * 1e3,
                 "compliance": comp, "levels": sizes}
                for lr, sizes, (rec, comp) in zip(runners, level_sizes, state["last"])]

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
    sens = sensitivity_roofline(args, w, K, L, law, rho_d, f_d, dc, roof["peak"])
    e2e = e2e_run(args, w, K, hs, L, law, world)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "setup_ms": setup_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json config %d)" % args.config,
            "config": config_dict(w, args, world), "leg_results": leg_results(),
            "roofline": roof, "sensitivity": sens, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ol = OracleLegs(w, threads=1)
        wk, dt = ol.step(1)
        line["cpu_baseline"] = {"value": wk / dt, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": "oracle port (numpy/scipy, 1 thread): one 1-iteration PCG solve + "
                                          "compliance + sensitivity per leg, %.1f s (after a %.0f s setup that is "
                                          "not part of the metric)" % (dt, ol.setup_s)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def _profile_summary():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
    except Exception:  # noqa: BLE001
        return {}


def roofline(args, w, state, L):
    """Dominant kernel of the config-4 PCG iteration: one level-0 Chebyshev step
    k_cheb<3, FineOp<3>> (4 of the 7 level-0 operator applications per
    iteration).  Algorithmic bytes per launch: reads r, D^-1, p, x and writes
    x, p', r' (7 x 8 B per dof), moduli (8 B per element) and free-dof masks
    (1 B per node); its launches stream from HBM (working set ~350 MB).  Timed
    with CUDA events around a CUDA graph of --roofline-reps back-to-back
    launches on the launching stream (tmg_hierarchy_time_smoother, level 0)."""
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
    check(L.tmg_hierarchy_time_smoother(h.handle, 0, args.roofline_reps, C.byref(ms),
                                        torch.cuda.current_stream().cuda_stream))
    mesh = w.mesh
    d = mesh.ndim
    nodes, nel = mesh.node_count, mesh.element_count
    cheb = w.solvers[0]["smoother"] == "chebyshev"
    nvec = 7 if cheb else 4
    bytes_launch = nodes * (nvec * 8 * d + 1) + nel * 8
    achieved = bytes_launch / (ms.value / 1e3) / 1e9
    prof = _profile_summary().get("config%d" % args.config, {})
    name = ("k_cheb<%d,FineOp<%d>> (level-0 Jacobi-Chebyshev step, matrix-free K)" % (d, d) if cheb
            else "k_jacobi<%d,FineOp<%d>> (level-0 weighted-Jacobi sweep, matrix-free K)" % (d, d))
    return {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": prof.get("dominant_dram_bytes"),
            "traffic_source": prof.get("source"), "bytes_per_launch": bytes_launch, "launch_us": ms.value * 1e3,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
            "timing": "CUDA events around one replay of a CUDA graph of %d back-to-back launches" % args.roofline_reps,
            "note": "working set %.0f MB vs 126 MB L2" % (bytes_launch / 1e6)}


def sensitivity_roofline(args, w, K, L, law, rho_d, f_d, dc, peak):
    """The fused compliance + sensitivity kernel k_sens (optimization.py:106-111,
    124-129): per launch it reads u and f (8 B per dof each), rho (8 B per
    element) and writes dc (8 B per element).  Timed as a CUDA graph of
    back-to-back launches rotating over three copies of u and f (HBM-fed)."""
    import torch
    from paper_2001_01655_b200._dev import as_dev, ptr
    from paper_2001_01655_b200._lib import check
    u = as_dev(np.random.default_rng(3).standard_normal(w.ndof))
    ms = C.c_double()
    reps = 3 * max(1, args.roofline_reps // 3)
    check(L.tmg_operator_time_sensitivity(K.handle, ptr(rho_d), ptr(f_d), ptr(u), law.penalty, law.e_max, law.e_min,
                                          ptr(dc), reps, C.byref(ms), torch.cuda.current_stream().cuda_stream))
    nbytes = 16 * w.ndof + 16 * w.mesh.element_count
    achieved = nbytes / (ms.value / 1e3) / 1e9
    return {"kernel": "k_sens<%d> (compliance f.u + per-element dc in one launch)" % w.mesh.ndim, "bound": "hbm",
            "launch_us": ms.value * 1e3, "bytes_per_launch": int(nbytes), "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak,
            "timing": "CUDA events around one replay of a CUDA graph of %d back-to-back launches rotating over 3 "
                      "copies of u and f" % reps}


def e2e_run(args, w, K, hs, L, law, world=1):
    """The same step through the public Python API with host buffers: the load
    vector from pinned host memory in (H2D), cg_solve + compliance_sensitivity,
    u and dc back to host memory (D2H) -- all inside the timed region."""
    import torch

    import paper_2001_01655_b200 as T
    from paper_2001_01655_b200 import _lib
    from paper_2001_01655_b200._dev import empty_dev, ptr, stream_ptr
    f_host = torch.from_numpy(np.ascontiguousarray(w.bc.load_vector)).pin_memory()
    rho_host = torch.from_numpy(np.ascontiguousarray(w.rho)).pin_memory()
    u_host = torch.empty(w.ndof, dtype=torch.float64).pin_memory()
    dc_host = torch.empty(w.mesh.element_count, dtype=torch.float64).pin_memory()
    rho_d = rho_host.cuda()
    dc = empty_dev(w.mesh.element_count)
    cfg = T.SolveConfig(method="cg", rtol=w.rtol, max_iterations=args.iters)

    def call():
        work = 0
        for h in hs:
            f_d = f_host.cuda(non_blocking=True)
            u, rec = T.cg_solve(K, f_d, None, h, cfg)
            comp = C.c_double()
            _lib.check(L.tmg_compliance_sensitivity(K.handle, ptr(rho_d), ptr(f_d), ptr(u), law.penalty,
                                                    law.e_max, law.e_min, ptr(dc), C.byref(comp),
                                                    stream_ptr(None)))
            u_host.copy_(u, non_blocking=True)
            dc_host.copy_(dc, non_blocking=True)
            torch.cuda.synchronize()
            work += w.ndof * rec.iterations
        return work
    call()
    work = secs = 0.0
    for _ in range(max(1, args.e2e_steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        work += call()
        secs += time.perf_counter() - t0
    h2d = len(hs) * f_host.numel() * 8
    d2h = len(hs) * (u_host.numel() + dc_host.numel()) * 8 + len(hs) * 8 * (args.iters + 1)
    ms, value = replica_throughput(1e3 * secs, work, world, "cuda")
    return {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": ms / max(1, args.e2e_steps),
            "timing": "host wall clock (synchronised) around the public-API step with host buffers: f H2D from "
                      "pinned memory, cg_solve, compliance_sensitivity, u and dc D2H (+ the residual history)"}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()

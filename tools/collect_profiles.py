"""Copy the round's gpurun_out/ artefacts into profiles/ (tracked): bench lines,
the ncu launch list of the bench command, digests of the ncu --set full captures
(details page + the raw metrics the roofline entries use) and the A/B tables.

    python tools/collect_profiles.py [--round r02]
"""
import argparse
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")

RAW = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "launch__shared_mem_per_block_dynamic", "launch__waves_per_multiprocessor",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"]


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, units, vals = rows[hdr], rows[hdr + 1], rows[hdr + 2]
    return {n: (vals[i], units[i]) for i, n in enumerate(h)}


def to_bytes(v, unit):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def digest(name, rnd):
    raw = os.path.join(G, "full_%s_%s.raw.csv" % (name, rnd))
    det = os.path.join(G, "full_%s_%s.details.txt" % (name, rnd))
    if not os.path.exists(raw):
        return None
    m = raw_metrics(raw)
    out = os.path.join(P, "%s_full_%s.txt" % (rnd, name))
    with open(out, "w") as fh:
        fh.write("# ncu --set full --clock-control none, one launch (tools/gpu_%s_profiles.sh); selected raw metrics, "
                 "then the details page\n" % rnd)
        for k in RAW:
            if k in m:
                fh.write("%-88s %s %s\n" % (k, m[k][0], m[k][1]))
        fh.write("\n")
        if os.path.exists(det):
            keep = [l for l in open(det) if not l.startswith("==PROF==")]
            fh.write("".join(keep))
    return m


def bench_json(log):
    if not os.path.exists(log):
        return None
    for line in open(log):
        if line.startswith("{"):
            return json.loads(line)
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r02")
    a = ap.parse_args()
    r = a.round
    os.makedirs(P, exist_ok=True)
    for src, dst in (("bench_%s.log" % r, "%s_bench_line.json" % r), ("bench_ref_%s.log" % r, "%s_bench_reference_line.json" % r)):
        d = bench_json(os.path.join(G, src))
        if d:
            json.dump(d, open(os.path.join(P, dst), "w"), indent=1)
    launches = os.path.join(G, "launches_bench_%s.csv" % r)
    if os.path.exists(launches):
        import ncu_summary
        shutil.copy(launches, os.path.join(P, "%s_launches_bench.csv" % r))
        with open(os.path.join(P, "%s_launches_bench.txt" % r), "w") as fh:
            fh.write("# TMG_PCG_EAGER=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv python bench.py "
                     "--steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1\n# (setup once + 3 two-iteration steps + the "
                     "roofline/sensitivity timing graphs + 2 e2e steps; per-launch times are cold-cache and serialised)\n")
            fh.write(ncu_summary.summary(launches, 60, 90) + "\n")
    summ_path = os.path.join(P, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for name in ("cheb3d_bench", "cheb3d", "residual3d", "cheb3d_stencil", "cgpq3d", "sens", "dgemm", "dgemm_gram", "gemv"):
        m = digest(name, r)
        if m and name == "cheb3d_bench":
            rd = to_bytes(*m["dram__bytes_read.sum"])
            wr = to_bytes(*m["dram__bytes_write.sum"])
            summ["config4"] = {"kernel": "k_cheb<3,FineOp<3>> (level-0 Jacobi-Chebyshev step, 3D matrix-free K)",
                               "dominant_dram_bytes": int(rd + wr), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
                               "ncu_duration_us": float(m["gpu__time_duration.sum"][0].replace(",", "")),
                               "source": "profiles/%s_full_cheb3d_bench.txt (ncu --set full of one launch of bench.py's own "
                                         "roofline timing graph: the same launch configuration, caches flushed by ncu)" % r}
        if m and name == "sens":
            rd = to_bytes(*m["dram__bytes_read.sum"])
            wr = to_bytes(*m["dram__bytes_write.sum"])
            summ["config4_sensitivity"] = {"kernel": "k_sens<3>", "dram_bytes": int(rd + wr),
                                           "source": "profiles/%s_full_sens.txt" % r}
    json.dump(summ, open(summ_path, "w"), indent=1)
    for src, dst in (("roofline_c1.txt", "%s_roofline_c1.txt"), ("roofline_c2.txt", "%s_roofline_c2.txt"),
                     ("roofline_c3.txt", "%s_roofline_c3.txt"), ("roofline_c4.txt", "%s_roofline_c4.txt"),
                     ("configs_%s.txt" % r, "%s_configs.txt"), ("setup_%s.txt" % r, "%s_setup.txt"),
                     ("iter_breakdown_c3.txt", "%s_iter_breakdown_c3.txt"), ("iter_breakdown_c4.txt", "%s_iter_breakdown_c4.txt"),
                     ("coarse_accuracy.txt", "%s_coarse_accuracy.txt"), ("c1_gmg_gap.log", "%s_c1_gmg_gap.txt"),
                     ("c1_gmg_gap2.log", "%s_c1_gmg_gap2.txt"), ("launches_chol_%s.csv" % r, "%s_launches_chol.csv")):
        if os.path.exists(os.path.join(G, src)):
            shutil.copy(os.path.join(G, src), os.path.join(P, dst % r))
    ck = os.path.join(G, "pytest_gpu_all.log")
    if os.path.exists(ck):
        with open(os.path.join(P, "%s_checkpoints.txt" % r), "w") as fh:
            fh.write("# python -m pytest tests -m gpu -q -s | grep 'k=' : device vs oracle at fixed iteration counts "
                     "(tests/test_gpu_configs.py); floor = the oracle against itself under rounding-level changes\n")
            fh.write("".join(l.lstrip(".F") for l in open(ck) if "k=" in l or "passed" in l or "failed" in l))
    print("profiles/ updated for", r)


if __name__ == "__main__":
    main()

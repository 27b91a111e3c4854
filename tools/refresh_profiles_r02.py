"""Copy one tools/gpu_evidence_r2.sh run (gpurun_out/ev, gpurun_out/*checked*)
into profiles/r02/ and regenerate its summaries: bench lines, the ncu summary
and profiles/ncu_traffic.json, the launch list, the DFMA counters, traces,
the SASS census and the checked-build record.  Prints the bench table rows.

  python tools/refresh_profiles_r02.py
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summarise  # noqa: E402

EV = os.path.join(ROOT, "gpurun_out", "ev")
DST = os.path.join(ROOT, "profiles", "r02")


def cp(src, dst):
    shutil.copy(os.path.join(EV, src), os.path.join(DST, dst))


out, traffic = {}, {}
for tag, rep, cfg in [("ring_c2", "prof_ring_c2", "config2"), ("ring_c3", "prof_ring_c3", "config3"),
                      ("ring_c4", "prof_ring_c4", "config4"), ("ring_c5", "prof_ring_c5", "config5"),
                      ("fin_c2", "prof_fin_c2", None)]:
    s = summarise(os.path.join(EV, rep + ".ncu-rep"))[0]
    out[tag] = s
    if cfg:
        traffic[cfg] = s["dram_read"] + s["dram_write"]
json.dump(out, open(os.path.join(DST, "ncu_summary.json"), "w"), indent=1)
traffic["source"] = ("profiles/r02/ncu_summary.json: dram__bytes_read.sum + dram__bytes_write.sum of one "
                     "ring_hull_kernel launch, ncu --set full --clock-control none (final round-2 code)")
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
for c in range(1, 6):
    cp(f"bench_c{c}.json", f"bench_c{c}.json")
for a, b in [("bench_reference_c4.json", "bench_reference_c4.json"), ("launches_c4.csv", "launches_config4.csv"),
             ("lscpu.txt", "lscpu.txt"), ("trace_ring.log", "trace_ring.log"), ("trace_fin_c2.log", "trace_finalize_c2.log"),
             ("steal_diag.log", "steal_diag.log"), ("time_dent.log", "time_dent.log")]:
    cp(a, b)
for c in (3, 4):
    lines = [l for l in open(os.path.join(EV, f"ncu_dfma_c{c}.log")) if l.strip().startswith(("void", "gpu__", "smsp__"))]
    open(os.path.join(DST, f"ncu_dfma_c{c}.txt"), "w").writelines(lines)
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_summary.py"), "--md", os.path.join(DST, "sass_summary.md")],
               cwd=ROOT, check=True, capture_output=True)
for k, s in out.items():
    print(k, s["kernel"][:50], round(s["duration"], 1), round(s["dram_read"] / 1e6, 1), round(s["dram_write"] / 1e6, 1),
          round(s["issue_active_pct"]), round(s["achieved_occupancy_pct"], 1), int(s["smem_ld_conflicts"]),
          round(s["warp_insts"] / 1e6, 1))
for c in range(1, 6):
    d = json.loads(open(os.path.join(DST, f"bench_c{c}.json")).read().strip().splitlines()[-1])
    r, e = d["roofline"], d["e2e"]
    print(f"| {c} | {d['config']['storage']} | {r['kernel_ms'] * 1e3:.1f} | {d['ms_per_step'] * 1e3:.1f} | {d['value']:.1f} | "
          f"{r['frac']:.3f} | {r['bare_read']['kernel_vs_bare_read']:.2f} | {e['value']:.2f} / {e['pageable']['value']:.2f} | "
          f"{d['cpu_baseline']['value']:.3f} |")

"""Summarise an ncu report (.ncu-rep) into the numbers the roofline and the
profiles/ notes cite: duration, DRAM bytes, throughput, occupancy, issue
activity, warp-stall breakdown, divergence and shared-memory conflicts.

  python tools/ncu_summary.py gpurun_out/prof_c2.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
    ("launch__registers_per_thread", "registers"),
    ("launch__occupancy_limit_shared_mem", "occ_limit_smem"),
    ("launch__occupancy_limit_registers", "occ_limit_regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_ld_conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem_st_conflicts"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma_thread_insts"),
]
STALL = "smsp__average_warps_issue_stalled_"


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit)
    return float(v) * scale if scale else float(v)


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        k = {"kernel": d.get("Kernel Name", "")}
        for key, name in KEYS:
            if key in d and d[key] != "":
                v = d[key].replace(",", "")
                try:
                    k[name] = to_bytes(v, u[key]) if name.startswith("dram_") and "pct" not in name else float(v)
                except ValueError:
                    k[name] = v
                if name == "duration":
                    k["duration_unit"] = u[key]
        stalls = {}
        for key in head:
            if key.startswith(STALL) and key.endswith("_per_issue_active.ratio"):
                try:
                    stalls[key[len(STALL):-len("_per_issue_active.ratio")]] = float(d[key])
                except ValueError:
                    pass
        k["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda t: -t[1])[:8])
        out.append(k)
    return out


def main():
    rep = sys.argv[1]
    res = summarise(rep)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)
    for k in res:
        print(json.dumps(k))


if __name__ == "__main__":
    main()

"""Turn a round's ncu outputs (gpurun_out/) into the committed summaries under
profiles/<round>/ plus profiles/ncu_traffic.json (bench.py's roofline.traffic).

  python tools/make_profiles.py r01
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summarise  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")


def launch_list(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    head = rows[0]
    k, v = head.index("Kernel Name"), head.index("Metric Value")
    per = defaultdict(list)
    for r in rows[1:]:
        if r[head.index("Metric Name")] == "gpu__time_duration.sum":
            per[r[k]].append(float(r[v].replace(",", "")))
    total = sum(sum(x) for x in per.values())
    res = []
    for name, xs in sorted(per.items(), key=lambda t: -sum(t[1])):
        res.append({"kernel": name[:120], "launches": len(xs), "mean_ns": sum(xs) / len(xs),
                    "share_of_listed_time": sum(xs) / total})
    return res


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    summary = {}
    ll = os.path.join(OUT, "launches_c2.csv")
    if os.path.exists(ll):
        summary["launch_list_config2"] = launch_list(ll)
    traffic = {}
    for tag, cfg in [("prof_ring_c2", "config2"), ("prof_ring_c5", "config5"), ("prof_ring_c4", "config4"),
                     ("prof_ring_c3", "config3"), ("prof_fin_c2", None)]:
        rep = os.path.join(OUT, tag + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        s = summarise(rep)
        summary[tag] = s
        if cfg:
            k = s[0]
            traffic[cfg] = k["dram_read"] + k["dram_write"]
    with open(os.path.join(dst, "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    old.update(traffic)
    with open(tpath, "w") as f:
        json.dump(old, f, indent=1)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    main()

"""SASS opcode census of libhood_b200.so per kernel (cuobjdump -sass): the
evidence that the double predicate never contracts into DFMA (geom.hpp:22-28,
SURVEY.md F3), where FFMA appears (the float filter's bound only), and which
memory paths each kernel uses (LDGSTS = cp.async, UTMALDG/UBLKCP = TMA /
bulk copies, LDS/STS widths).

  python tools/sass_summary.py [lib.so] [--md out.md]
"""
import collections
import re
import subprocess
import sys

so = next((a for a in sys.argv[1:] if a.endswith(".so")), "paper_1203_5004_b200/lib/libhood_b200.so")
out_md = sys.argv[sys.argv.index("--md") + 1] if "--md" in sys.argv else None
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in txt.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(\.[A-Z0-9_]+)*)", line)
    if m and cur:
        op = m.group(2)
        funcs[cur][op] += 1
        funcs[cur][op.split(".")[0] + "*"] += 1

WATCH = ["DFMA*", "DMUL*", "DADD*", "DSETP*", "FFMA*", "FMUL*", "FADD*", "LDGSTS*", "UTMALDG*", "UBLKCP*", "SYNCS*",
         "LDG*", "STG*", "LDS*", "STS*", "SHFL*", "REDUX*", "CREDUX*", "VOTE*", "ATOMG*", "RED*", "BAR*", "CALL*"]


def short(name):
    m = re.search(r"hood_b200(\d+)([a-z_]+?)(I[fd])?", name)
    base = re.sub(r"^_ZN9hood_b200\d+", "", name)
    base = re.sub(r"EEEv.*|EEv.*|Ev.*", "", base)
    return base[:60]


rows = []
for f, c in funcs.items():
    rows.append((short(f), {k: c.get(k, 0) for k in WATCH}, {k: v for k, v in c.items() if k.startswith(("LDS.", "STS.", "LDG.", "STG."))}))
hdr = "| kernel | " + " | ".join(w.rstrip("*") for w in WATCH) + " |"
lines = [hdr, "|" + "---|" * (len(WATCH) + 1)]
for name, w, _ in rows:
    lines.append(f"| `{name}` | " + " | ".join(str(w[k]) for k in WATCH) + " |")
text = "\n".join(lines)
print(text)
if out_md:
    with open(out_md, "w") as fh:
        fh.write("# SASS opcode census (cuobjdump -sass of " + so + ", sm_100a)\n\n")
        fh.write("Static instruction counts per kernel (device functions inlined or called from the kernel are "
                 "included in its listing).  DFMA = 0 everywhere: the reference's orient is evaluated with separately "
                 "rounded __dmul_rn/__dsub_rn (geom.hpp:22-28), never contracted.\n\n")
        fh.write(text + "\n\nMemory opcode widths:\n\n")
        for name, _, widths in rows:
            fh.write(f"- `{name}`: " + ", ".join(f"{k} {v}" for k, v in sorted(widths.items())) + "\n")

"""Per-role instruction / stall-sample split of the stream kernel from an ncu source page
(ncu -i rep --page source --csv --print-source=cuda,sass > src.csv; python tools/ncu_roles.py src.csv).
SASS instructions are assigned to the warp role of the nearest preceding stream.cu line."""
import csv
import sys

src_lines = open("paper_2105_05879_b200/csrc/stream.cu").read().splitlines()


def find(pat):
    for i, l in enumerate(src_lines):
        if pat in l:
            return i + 1
    raise SystemExit(f"marker not found: {pat}")


marks = sorted([(find("// ======================= producer"), "producer"),
                (find("// ======================= coefficient"), "coefficient"),
                (find("// ======================= tail warps"), "tail"),
                (find("// ---- refinement: v_i = a_i . x"), "tail:refinement"),
                (find("// ======================= consumer"), "consumer"),
                (find("// ----------------------------------------------------------- refinement ----"), "tail:refinement"),
                (find("// --------------------------------------------------------------- kernel ----"), "kernel"),
                (find("__device__ __forceinline__ float coef_"), "coefficient") if any("float coef_" in l for l in src_lines) else (0, "pre")])


def role(line):
    r = None
    for ln, name in marks:
        if line >= ln:
            r = name
    return r


cur = hdr = None
insts = []
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] in ("Function Name",):
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and cur and len(r) == len(hdr) and not r[0].isdigit() and r[2].startswith("0x"):
        d = dict(zip(hdr, r))
        insts.append((int(r[2], 16), cur, lineno, r[3].strip(), float(d["Instructions Executed"] or 0),
                      float(d["Warp Stall Sampling (All Samples)"] or 0)))
    elif hdr and cur and len(r) == len(hdr) and r[0].isdigit():
        lineno = int(r[0])
insts.sort()
tot = sum(i[4] for i in insts) or 1
ts = sum(i[5] for i in insts) or 1
last = "?"
agg, spin = {}, {}
for a, f, l, s, c, smp in insts:
    if f == "stream.cu":
        last = role(l) or last
    agg.setdefault(last, [0, 0])
    agg[last][0] += c
    agg[last][1] += smp
    if "SYNCS.PHASECHK" in s or "NANOSLEEP" in s or (f == "fst_common.cuh" and "BRA" in s):
        spin[last] = spin.get(last, 0) + c
print(f"total {tot:.3e} warp-instructions, {ts:.0f} stall samples")
for k, (c, smp) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:18s} inst {100 * c / tot:5.1f}%  (mbarrier wait loop {100 * spin.get(k, 0) / tot:4.1f}%)  stall samples {100 * smp / ts:5.1f}%")

"""Summarise an .ncu-rep (raw metrics + top source lines by stall samples) into text."""
import csv
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    print(f"# {rep}\nkernel: {v[h.index('Kernel Name')] if 'Kernel Name' in h else '?'}")
    for name in METRICS:
        if name in h:
            i = h.index(name)
            print(f"{name:70s} {v[i]:>22s} {u[i]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, out = None, None, []
    for r in csv.reader(src.splitlines()):
        if r and r[0] == "File Path":
            cur = r[1]
            continue
        if r and r[0] == "Function Name":
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and cur and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                inst = float(d["Instructions Executed"] or 0)
                samp = float(d["Warp Stall Sampling (All Samples)"] or 0)
            except ValueError:
                continue
            if d["Line No"].isdigit():
                out.append((samp, inst, cur.split("/")[-1], d["Line No"], d))
    tot_s = sum(o[0] for o in out) or 1
    tot_i = sum(o[1] for o in out) or 1
    stalls = [k for k in (hdr or []) if k.startswith("stall_") and "Not Issued" not in k]
    print("\ntop source lines by warp-stall samples:")
    for o in sorted(out, key=lambda x: -x[0])[:15]:
        top = sorted(((float(o[4][k] or 0), k) for k in stalls), reverse=True)[:3]
        print(f"{100 * o[0] / tot_s:5.1f}% samples {100 * o[1] / tot_i:5.1f}% inst  {o[2]}:{o[3]}  "
              f"{[(k[6:], int(val)) for val, k in top]}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Summarise an ncu source page: stall samples by SASS opcode and reason."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
iS = hdr.index("Warp Stall Sampling (All Samples)")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.Counter()
st = collections.Counter()
reasons = collections.Counter()
for r in data:
    toks = r[1].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    agg[op] += int(r[iS])
    for i in cols:
        st[(op, hdr[i])] += int(r[i])
        reasons[hdr[i]] += int(r[i])
tot = sum(agg.values()) or 1
print("reasons:", [(k, round(100 * v / tot, 1)) for k, v in reasons.most_common(8)])
for op, c in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    top = sorted([(v, k[1]) for k, v in st.items() if k[0] == op], reverse=True)[:3]
    print(f"{op:14s} {100 * c / tot:5.1f}%  {top}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rr = list(csv.reader(raw))
want = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct")
for k in range(2, len(rr)):
    print({h: (u, v) for h, u, v in zip(rr[0], rr[1], rr[k]) if h in want})

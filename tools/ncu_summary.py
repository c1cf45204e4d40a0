"""Summarise an ncu --set full report: per launch duration, DRAM bytes, DRAM %, tensor-pipe activity, grid, regs
(markdown table).  Usage: python tools/ncu_summary.py REPORT.ncu-rep"""
import csv, subprocess, sys
mets = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__registers_per_thread"]
f = sys.argv[1]
out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv", "--metrics", ",".join(mets)], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]; units = r[1]
idx = {k: i for i, k in enumerate(h)}
print("| kernel | µs | DRAM read MB | DRAM write MB | DRAM % peak | tensor pipe active % | grid | regs |")
print("|---|---|---|---|---|---|---|---|")
for row in r[2:]:
    name = row[idx["Kernel Name"]].split("(")[0].replace("void ", "")
    g = lambda m: row[idx[m]] if m in idx else "?"
    def mb(m):
        v = float(g(m)); u = units[idx[m]]
        return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
    def us(m):
        v = float(g(m)); u = units[idx[m]]
        return v * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
    print(f"| `{name}` | {us(mets[0]):.1f} | {mb(mets[1]):.1f} | {mb(mets[2]):.1f} | {float(g(mets[3])):.1f} | {float(g(mets[4])):.1f} | {g(mets[5])} | {g(mets[6])} |")

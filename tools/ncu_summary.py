"""Summarise an ncu --set full report of run_kernel into profiles/.
usage: python tools/ncu_summary.py gpurun_out/prof_run.ncu-rep profiles/r01_run_kernel"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
def page(p, extra=()):
    return subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra],
                          capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(page("raw"))))
hdr, units, vals = raw[0], raw[1], raw[2]
R = dict(zip(hdr, vals))
U = dict(zip(hdr, units))
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct"]
lines = []
res = {}
for k in want:
    if k in R:
        lines.append(f"{k:80s} {R[k]} {U.get(k, '')}")
        res[k] = R[k]
stalls = sorted(((float(v.replace(",", "")), h) for h, v in zip(hdr, vals)
                 if "pcsamp_warps_issue_stalled" in h and h.endswith("not_issued")
                 and v.replace(",", "").replace(".", "").isdigit()), reverse=True)[:10]
lines.append("\nwarp stall samples (not issued):")
lines += [f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {v:.0f}" for v, h in stalls]
src = page("source", ("--print-source", "sass"))
hist = subprocess.run([sys.executable, "tools/sass_hist.py"], input=src, capture_output=True,
                      text=True).stdout
regions = subprocess.run([sys.executable, "tools/sass_regions.py", "8"], input=src,
                         capture_output=True, text=True).stdout
open(out + ".txt", "w").write("\n".join(lines) + "\n\nSASS opcode mix (executed warp instructions):\n"
                               + hist + "\nhottest straight-line regions:\n" + regions)
try:
    res["dram_bytes_per_launch"] = float(R["dram__bytes_read.sum"].replace(",", "")) + \
        float(R["dram__bytes_write.sum"].replace(",", ""))
    # ncu reports in the unit of the column (byte/Kbyte/Mbyte/Gbyte)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res["dram_bytes_per_launch"] = sum(float(R[k].replace(",", "")) * scale.get(U[k], 1)
                                       for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
except KeyError:
    pass
json.dump(res, open(out + ".json", "w"), indent=1)
print(open(out + ".txt").read())

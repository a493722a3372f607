"""Summarise an ncu report (one capture per kernel launch) into a JSON +
markdown table: duration, DRAM bytes, issue utilisation, pipe utilisation
(FP32 FMA / ALU / XU / FP64, % of peak over active cycles), occupancy, SM
active/elapsed.  Usage: python tools/ncu_summary.py rep.ncu-rep out_prefix"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_active.avg",
           "gpc__cycles_elapsed.max", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "smsp__inst_executed.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           # pipe utilisation (issue-bound kernels): FP32 FMA, ALU, XU (MUFU /
           # conversions), FP64
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def main(rep, prefix):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))

        def f(k):
            return float(d[k].replace(",", ""))
        t = f("gpu__time_duration.sum")
        t_us = t / 1e3 if u["gpu__time_duration.sum"] == "ns" else (t if u["gpu__time_duration.sum"] == "us" else t * 1e3)

        def b(k):
            v = f(k)
            s = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[k], 1)
            return v * s
        res.append({"kernel": d["Kernel Name"], "duration_us": t_us,
                    "dram_read_bytes": b("dram__bytes_read.sum"),
                    "dram_write_bytes": b("dram__bytes_write.sum"),
                    "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "sm_active_over_elapsed": f("sm__cycles_active.avg") / max(f("gpc__cycles_elapsed.max"), 1),
                    "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
                    "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                    "regs": int(f("launch__registers_per_thread")),
                    "warp_inst": f("smsp__inst_executed.sum"),
                    "pipe_pct": {"fma": f("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                                 "alu": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                                 "xu": f("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                                 "fp64": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")}})
    with open(prefix + ".json", "w") as fh:
        json.dump({"source": rep, "note": "ncu --set full --clock-control none (cold, serialised)",
                   "kernels": res}, fh, indent=1)
    with open(prefix + ".md", "w") as fh:
        fh.write("| kernel | us | DRAM R MB | DRAM W MB | issue % | FMA / ALU / XU / FP64 pipe % "
                 "| SM active/elapsed | warps % | regs |\n")
        fh.write("|---|---|---|---|---|---|---|---|---|\n")
        for x in res:
            pp = x["pipe_pct"]
            fh.write(f"| {x['kernel'][:60]} | {x['duration_us']:.1f} | {x['dram_read_bytes']/1e6:.1f} | "
                     f"{x['dram_write_bytes']/1e6:.1f} | {x['issue_active_pct']:.1f} | "
                     f"{pp['fma']:.0f} / {pp['alu']:.0f} / {pp['xu']:.0f} / {pp['fp64']:.0f} | "
                     f"{x['sm_active_over_elapsed']:.2f} | {x['warps_active_pct']:.1f} | {x['regs']} |\n")
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

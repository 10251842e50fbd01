"""Summarise an .ncu-rep (speed of light, memory, stalls, top SASS lines)."""
import csv, io, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return [dict(zip(r[0], row)) for row in r[2:]], dict(zip(r[0], r[1]))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active"]

def main(rep):
    rows, units = raw(rep)
    for d in rows:
        print("kernel:", d.get("Kernel Name", "")[:80])
        for k in KEYS:
            if k in d:
                print(f"  {k:60s} {d[k]:>16s} {units.get(k,'')}")
        st = {k: float(v.replace(',', '')) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v not in ("", "n/a")}
        tot = sum(st.values()) or 1
        for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]:
            print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_',''):28s} {100*v/tot:5.1f}%")

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        main(rep)

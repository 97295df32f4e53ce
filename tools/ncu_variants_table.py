"""Summarise gpurun_out/m_<mf>.csv written by tools/ncu_variants.sh."""
import csv
import io
import sys

for mf in sys.argv[1:] or ["3", "2", "0"]:
    txt = open(f"gpurun_out/m_{mf}.csv").read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    agg = {}
    for r in rows:
        k = r["Kernel Name"].split("(")[0][-28:]
        agg.setdefault(k, {}).setdefault(r["Metric Name"], []).append(float(r["Metric Value"].replace(",", "")))
    print("matrix_free", mf)
    for k, v in agg.items():
        m = {a: sum(b) / len(b) for a, b in v.items()}
        print(f"  {k:30s} t={m['gpu__time_duration.sum']/1000:6.2f}us active={m['sm__cycles_active.avg']:7.0f} "
              f"elapsed={m['sm__cycles_elapsed.avg']:7.0f} inst={m['smsp__inst_executed.sum']/1e6:5.2f}M "
              f"warps%={m['sm__warps_active.avg.pct_of_peak_sustained_active']:5.1f} "
              f"issue%={m['smsp__issue_active.avg.pct_of_peak_sustained_active']:5.1f} "
              f"lsb={m['smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio']:5.2f} "
              f"L2MB={m['lts__t_bytes.sum']/1e6:6.1f} regs={m['launch__registers_per_thread']:.0f} "
              f"grid={m['launch__grid_size']:.0f}")

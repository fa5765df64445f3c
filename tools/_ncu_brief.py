"""Brief counters + top stall lines from ncu raw/source CSV pairs (profiling helper):
python tools/_ncu_brief.py gpurun_out/ncu_<kernel>_<n>   (prefix of _raw.csv / _source.csv)"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__cluster_dim_x"]
for pre in sys.argv[1:]:
    rows = list(csv.reader(open(pre + "_raw.csv")))
    if len(rows) < 3:
        print(pre, "empty")
        continue
    h, u = rows[0], rows[1]
    print("==", pre, rows[2][h.index("Kernel Name")][:80])
    for k in KEYS:
        if k in h:
            print("   %-70s %s %s" % (k, rows[2][h.index(k)], u[h.index(k)]))
    try:
        src = list(csv.reader(open(pre + "_source.csv")))
    except FileNotFoundError:
        continue
    sh, data = src[1], src[2:]
    iS = sh.index("Warp Stall Sampling (All Samples)")
    stalls = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(float(r[iS]) for r in data) or 1
    agg = {c: sum(float(r[sh.index(c)]) for r in data) for c in stalls}
    print("   stalls:", ", ".join("%s %.0f%%" % (c[6:], 100 * v / tot) for c, v in sorted(agg.items(), key=lambda x: -x[1])[:6]))
    for r in sorted(data, key=lambda r: -float(r[iS]))[:12]:
        print("   %6.1f%% %s %s" % (100 * float(r[iS]) / tot, r[0][-5:], r[1].strip()[:60]))

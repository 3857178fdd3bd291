"""Key metrics of an ncu report (one kernel): python tools/ncu_summary.py file.ncu-rep"""
import csv, io, subprocess, sys
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.max"]
for f in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, zip(vals, units)))
    print(f, "|", d.get("Kernel Name", ("?",))[0][:70])
    for k in WANT:
        if k in d:
            print(f"  {k:75s} {d[k][0]:>16s} {d[k][1]}")
    for k in hdr:
        if "tensor" in k and k not in WANT and ".avg.pct" in k and "ops_path" not in k and d[k][0] not in ("0", ""):
            print(f"  {k:75s} {d[k][0]:>16s} {d[k][1]}")

"""Summarise ncu --set full captures (gpurun_out/*.ncu-rep) into profiles/:
a markdown table of the counters the roofline claims rest on, and
profiles/ncu_traffic.json (dram bytes per launch) that bench.py reports as
roofline.traffic.  usage: python tools/ncu_summary.py OUT.md rep:key [rep:key ...]
(key = "<kernel family>/n<n>/<dtype>" as bench.py looks it up)."""
import csv, io, json, subprocess, sys
from pathlib import Path

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:       # empty capture (kernel filter matched nothing)
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def main():
    out_md = Path(sys.argv[1])
    import os
    traffic_path = Path(os.environ.get("NCU_TRAFFIC_JSON", "profiles/ncu_traffic.json"))
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    lines = [f"# ncu --set full captures ({out_md.stem})", "",
             "`ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 2 -c 1`"
             " on one B200 (cold L2, serialised replay: absolute times are not bench times).", ""]
    for arg in sys.argv[2:]:
        rep, key = arg.split(":", 1)
        d = raw(rep)
        if d is None:
            lines += [f"## {key}  ({Path(rep).name})", "", "(no kernel captured)", ""]
            continue
        name = d.get("Kernel Name", ("?", ""))[0]
        lines += [f"## {key}  ({Path(rep).name})", "", f"kernel: `{name[:160]}`", "", "```"]
        for m in METRICS:
            if m in d:
                v, u = d[m]
                lines.append(f"{m:100s} {v} {u}")
        lines += ["```", ""]
        def mb(m):
            v, u = d[m]
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        if "dram__bytes_read.sum" in d:
            traffic[key] = int(mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"))
    out_md.write_text("\n".join(lines))
    traffic_path.write_text(json.dumps(traffic, indent=1, sort_keys=True))
    print(out_md, traffic)


if __name__ == "__main__":
    main()

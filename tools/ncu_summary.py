"""Summarise ncu captures into profiles/ (markdown + json).  Usage:
python tools/ncu_summary.py OUT_PREFIX name=path.ncu-rep [...] [--launches launches.csv]"""
import csv, io, json, subprocess, sys, collections
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__cycles_elapsed.avg.per_second", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
           "lts__t_sector_hit_rate.pct", "launch__shared_mem_per_block_dynamic"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3,
        "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}
out, args = sys.argv[1], sys.argv[2:]
md, js = [], {}
launches = None
if "--launches" in args:
    i = args.index("--launches"); launches = args[i + 1]; args = args[:i] + args[i + 2:]
for a in args:
    name, path = a.split("=", 1)
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for j, v in enumerate(rows[2:]):  # one row per captured launch
        kern = v[h.index("Kernel Name")]
        key = name if len(rows) == 3 else f"{name}[{j}]"
        md.append(f"## {key}: {kern[:90]}  ({path.split('/')[-1]}, ncu --set full --clock-control none, one launch)")
        d = {"kernel": kern}
        for m in METRICS:
            if m in h:
                k = h.index(m)
                md.append(f"- {m}: {v[k]} {units[k]}")
                try:
                    d[m] = float(v[k].replace(",", "")) * UNIT.get(units[k], 1)
                except ValueError:
                    d[m] = v[k]
        if "dram__bytes_read.sum" in d:
            d["dram_bytes_per_launch"] = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
            d["dram_gbs"] = d["dram_bytes_per_launch"] / d["gpu__time_duration.sum"] / 1e9
            md.append(f"- derived: DRAM traffic {d['dram_bytes_per_launch']/1e6:.1f} MB/launch, "
                      f"{d['dram_gbs']:.0f} GB/s over the (cold, serialised) launch")
        js[key] = d
        md.append("")
if launches:
    rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(x) for x in agg.values())
    md.append(f"## launch list ({launches.split('/')[-1]}): {sum(len(x) for x in agg.values())} launches of our kernels")
    md.append("| kernel | launches | mean us | share of our device time |")
    md.append("|---|---|---|---|")
    shares = {}
    for k, x in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        md.append(f"| {k} | {len(x)} | {sum(x)/len(x)/1e3:.2f} | {sum(x)/tot:.3f} |")
        shares[k] = sum(x) / tot
    js["launch_shares"] = shares
open(out + ".md", "w").write("\n".join(md) + "\n")
json.dump(js, open(out + ".json", "w"), indent=1)
print("\n".join(md))

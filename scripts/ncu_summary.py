"""Summaries of ncu output for profiles/ (committed evidence).

  python scripts/ncu_summary.py launches <launches.csv> <steps> <header>
      -> per-kernel launch table (avg us, launches, share of the step's kernel time)
  python scripts/ncu_summary.py raw <raw.csv> <header>
      -> per-kernel key metrics from an `ncu --set full` capture (--page raw --csv)
  python scripts/ncu_summary.py traffic <raw.csv> <source tag>
      -> profiles/ncu_traffic.json body (dram bytes per launch per kernel class)
"""
import csv
import json
import sys
from collections import defaultdict

CLASSES = {"k_sample": "sample", "k_fwd_tc": "field_fwd", "k_fwd_ws": "field_fwd", "k_fwd_ts": "field_fwd", "k_fwd_wx": "field_fwd",
           "k_fwd_tile": "field_fwd", "k_composite": "composite",
           "k_bwd_tc": "mlp_bwd", "k_bwd_tile": "mlp_bwd", "k_encode_bwd": "encode_bwd", "k_adam": "adam",
           "k_adam_fused": "adam"}

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "lts__t_sectors_srcunit_tex_op_red.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "lts__t_sectors.sum"]


def short(name):
    n = name.split("(")[0]
    return n.replace("(anonymous namespace)::", "")


def launches(path, steps, header):
    per = defaultdict(list)
    for r in csv.reader(open(path)):
        if len(r) < 15 or r[0] == "ID" or r[12] != "gpu__time_duration.sum":
            continue
        per[short(r[4])].append(float(r[14]) / 1e3)
    step_kernels = {k: v for k, v in per.items() if len(v) == steps}
    tot = sum(sum(v) for v in step_kernels.values()) or 1.0
    print(header)
    print("#   avg per launch launches share of step  kernel")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        share = f"{100 * sum(v) / tot:10.1f}%" if k in step_kernels else " " * 11
        print(f"{sum(v) / len(v):12.1f} us {len(v):8d} {share}  {k}")


def raw_rows(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    for r in rows[2:]:
        if len(r) == len(hdr):
            yield dict(zip(hdr, r)), dict(zip(hdr, rows[1]))


def raw(path, header, l2_peak_gbs=None):
    print(header)
    for d, u in raw_rows(path):
        print(f"\n{short(d['Kernel Name'])}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>18s} {u.get(k, '')}")
        if "lts__t_sectors.sum" in d:  # L2 bytes and rate (32 B sectors)
            t = float(d["gpu__time_duration.sum"].replace(",", "")) * (1e-3 if u["gpu__time_duration.sum"] == "ns" else 1)
            b = float(d["lts__t_sectors.sum"].replace(",", "")) * 32
            rate = b / (t * 1e-6) / 1e9
            line = f"  {'L2 bytes (lts__t_sectors x 32) / rate':70s} {b / 1e6:>14.1f} MB {rate:>9.1f} GB/s"
            if l2_peak_gbs:
                line += f"  ({rate / l2_peak_gbs:.2f} of the measured L2 peak {l2_peak_gbs:.0f} GB/s)"
            print(line)


def traffic(path, tag):
    out = {"_source": tag}
    for d, u in raw_rows(path):
        name = short(d["Kernel Name"])
        base = name.split("::")[-1].split("<")[0]
        cls = CLASSES.get(base)
        if not cls:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = sum(float(d[k].replace(",", "")) * scale.get(u[k], 1)
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        t = float(d["gpu__time_duration.sum"].replace(",", "")) * (1e-3 if u["gpu__time_duration.sum"] == "ns" else 1)
        out[cls] = {"kernel": name.split("::")[-1], "dram_bytes_per_launch": int(b), "gpu_time_us": round(t, 1)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    elif mode == "raw":
        raw(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
    else:
        traffic(sys.argv[2], sys.argv[3])

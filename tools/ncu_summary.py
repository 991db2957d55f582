"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv> <out.md>
    python tools/ncu_summary.py full <report.ncu-rep> <out.md> <out.json>

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list per
kernel (cold-cache, serialised: compare shares, not absolutes).  `full`
extracts the roofline-relevant metrics of a `--set full` capture and writes
the per-launch DRAM traffic JSON bench.py reports as `roofline.traffic`.
"""

import collections
import csv
import json
import subprocess
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
        "second": 1e3}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        name = r[ki].split("(")[0].replace("rs::<unnamed>::", "").replace("(anonymous namespace)::", "")
        if "at::" in name or "at_cuda_detail" in name:  # torch's own kernels (the synthetic-data generator)
            continue
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * UNIT[r[ui]])
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list: `{path.split('/')[-1]}`", "",
             "Cold-cache, serialised per-launch device times (`gpu__time_duration.sum`) of the library's kernels "
             "(torch's data-generator kernels dropped); compare shares.", "",
             "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v):.3f} | {100 * sum(v) / tot:.2f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
]


def full(rep, out_md, out_json):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    kname = m.get("Kernel Name", ("?", ""))[0]
    lines = [f"# ncu --set full: `{rep.split('/')[-1]}`", "", f"kernel: `{kname}`", "", "| metric | value | unit |",
             "|---|---:|---|"]
    for w in WANT:
        if w in m:
            lines.append(f"| `{w}` | {m[w][0]} | {m[w][1]} |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))

    def to_bytes(key):
        v, u = m[key]
        return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]

    js = {"kernel": kname, "report": rep.split("/")[-1],
          "dram_bytes_per_launch": to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum"),
          "duration_ms": float(m["gpu__time_duration.sum"][0].replace(",", "")) *
          UNIT.get(m["gpu__time_duration.sum"][1], 1.0),
          "tensor_pipe_pct": float(m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"][0]),
          "sm_clock_ghz": float(m["sm__cycles_elapsed.avg.per_second"][0])}
    json.dump(js, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4])

"""Summarise an ncu report (key throughput metrics + stall reasons) or an ncu launch list
(per-kernel share of device time) into a small text file for profiles/."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "gpc__cycles_elapsed.max", "sm__cycles_active.avg",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u = r[0], r[1]
    out = []
    for row in r[2:]:
        d = dict(zip(h, row))
        out.append(f"kernel: {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:70s} {d[k]} {u[h.index(k)]}")
        st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled")
              and not k.endswith("not_issued") and v.replace(".", "", 1).isdigit()]
        tot = sum(v for _, v in st) or 1.0
        for k, v in sorted(st, key=lambda x: -x[1])[:8]:
            out.append(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f} %")
    return "\n".join(out)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                     "second": 1e3, "s": 1e3}.get(d["Metric Unit"], 1.0)
            v = float(d["Metric Value"].replace(",", "")) * scale
            k = d["Kernel Name"].split("(")[0][:70]
            agg[k][0] += 1
            agg[k][1] += v
    tot = sum(v for _, v in agg.values()) or 1.0
    lines = [f"{'launches':>8} {'ms':>10} {'share':>7}  kernel"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{c:8d} {t:10.3f} {100 * t / tot:6.1f}%  {k}")
    return "\n".join(lines)


def traffic(path):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes) of the first kernel in a --set full report."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u = r[0], r[1]
    d, du = dict(zip(h, r[2])), dict(zip(h, u))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(d[k].replace(",", "")) * scale.get(du[k], 1)
    return tot


if __name__ == "__main__":
    # ncu_summary.py report|launches <file>
    # ncu_summary.py traffic <out.json> name=<report> ...   (per-launch DRAM bytes for bench.py)
    kind = sys.argv[1]
    if kind == "traffic":
        import json
        out = {}
        for a in sys.argv[3:]:
            name, path = a.split("=", 1)
            out[name] = traffic(path)
        json.dump(out, open(sys.argv[2], "w"), indent=1)
        print(out)
    else:
        path = sys.argv[2]
        print(report(path) if kind == "report" else launches(path))

"""Condense ncu output into the summaries kept under profiles/.

    python tools/ncu_summary.py launches <launches.csv>            # per-kernel share of a launch list
    python tools/ncu_summary.py report <x.ncu-rep> [flops_per_launch]  # key counters of one captured kernel

Runs here (no GPU): `ncu -i` reads the report.
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__average_warp_latency_per_inst_issued.ratio",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]
STALLS = ["wait", "math_pipe_throttle", "long_scoreboard", "short_scoreboard", "barrier", "selected",
          "not_selected", "membar", "branch_resolving", "mio_throttle", "lg_throttle", "no_instructions",
          "dispatch_stall"]


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("ddk::", "")
        if "at::" in name or "c10" in name or "cutlass" in name:
            name = "[harness] " + name[:40]
        tot[name] += v
        cnt[name] += 1
    ours = sum(v for k, v in tot.items() if not k.startswith("[harness]"))
    out = [f"{'kernel':44s} {'launches':>8s} {'ms':>10s} {'share of ours':>14s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        share = "" if k.startswith("[harness]") else f"{100 * v / ours:13.1f}%"
        out.append(f"{k:44s} {cnt[k]:8d} {v / 1e6:10.1f} {share:>14s}")
    return "\n".join(out)


def report(path, flops=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, row)}
        name = d.get("Kernel Name", ("?", ""))[0]
        out.append(f"kernel: {name[:120]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:78s} {d[k][0]} {d[k][1]}")
        tot = 0.0
        st = {}
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in d:
                try:
                    st[s] = float(d[k][0].replace(",", ""))
                    tot += st[s]
                except ValueError:
                    pass
        if tot:
            out.append("  stall samples: " + ", ".join(f"{s} {100 * v / tot:.1f}%" for s, v in
                                                       sorted(st.items(), key=lambda x: -x[1]) if v))
        try:
            t = float(d["gpu__time_duration.sum"][0].replace(",", ""))
            tunit = d["gpu__time_duration.sum"][1]
            tsec = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(tunit, 1e-9)
            rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) if "dram__bytes_read.sum" in d else 0
            out.append(f"  duration {tsec * 1e3:.3f} ms")
            if flops:
                out.append(f"  achieved {float(flops) / tsec / 1e12:.2f} TFLOP/s (algorithmic flops {float(flops):.3g})")
        except (KeyError, ValueError):
            pass
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None))

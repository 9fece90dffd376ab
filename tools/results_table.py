#!/usr/bin/env python
"""Render the BASELINE.md §4 results table from the round's bench lines (profiles/r02_bench_*.json)
and the full-size parity records (profiles/r02_fullsize_parity_*.json).

    python tools/results_table.py profiles/r02_bench_cfg0.json ... > /tmp/table.md
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(path):
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    return None


def fmt(x, f="{:.3g}"):
    return "—" if x is None else f.format(x)


def main(paths):
    rows = []
    par = {}
    for c in ("cfg2", "cfg3"):
        p = os.path.join(ROOT, "profiles", f"r02_fullsize_parity_{c}.json")
        if os.path.exists(p):
            par[c] = json.load(open(p))
    for path in paths:
        d = load(path)
        if not d or "roofline" not in d or d.get("impl") == "reference":
            continue
        name = os.path.basename(path).replace("r02_bench_", "").replace(".json", "")
        acc = d.get("accuracy", {})
        cb = d.get("cpu_baseline") or {}
        fp = par.get(name)
        rows.append("| {} | {} | {} | {} | {} | {} | {} | {} / {} | {} | {} | {} | {} | {} |".format(
            name, d["config"].get("n", "—"), fmt(d.get("factor_ms"), "{:.1f}"), fmt(d.get("value"), "{:.0f}"),
            fmt(100 * d["factor_frac_of_fp64_peak"] if d.get("factor_frac_of_fp64_peak") else None, "{:.1f}%"),
            fmt(d.get("solve_ms_per_batch"), "{:.1f}"), fmt(d.get("solve_ms_per_1000_rhs"), "{:.0f}"),
            fmt(acc.get("berr_max"), "{:.1e}"), fmt(acc.get("berr_unrefined_max"), "{:.1e}"),
            fmt(fp["rel_diff_max"], "{:.1e}") if fp else "corner samples (tests)",
            "yes (GPU == oracle)" if (fp and fp.get("gpu", {}).get("inertia") is not None) else
            ("—" if d["dtype"] == "c128" else "tests"),
            fmt(fp["oracle"]["factor_s"], "{:.0f} s (full)") if fp else fmt(cb.get("value"), "{:.0f} GFLOP/s (sample)"),
            fmt(cb.get("solve_ms_per_1000_rhs"), "{:.0f} ms/1000 (sample)"), cb.get("cores", "—")))
    print("| Config | n | Factor ms | Factor GFLOP/s | % of measured FP64 peak | Solve ms per batch | "
          "Solve ms per 1000 RHS | berr refined / unrefined | rel. diff vs oracle | Inertia equal | "
          "Oracle factor | Oracle solve | Oracle cores |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(r)


if __name__ == "__main__":
    main(sys.argv[1:])

"""M1: measured FP64 / complex128 GEMM peak on this B200 (cuBLAS via torch.matmul).

This is the denominator of every FP64 roofline fraction:
MEASURED_PEAKS.json carries only HBM and bf16 numbers.  Burst = best of 10 single
8192^3 products; sustained = back-to-back products for ~4 s.  Clocks sampled via
nvidia-smi during the sustained loop.  Writes JSON to stdout (and --out).
"""
import argparse, json, os, subprocess, time
import torch


def bench(dtype, n, reps_burst=10, sustain_s=4.0):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    flop = 2.0 * n ** 3 * (4 if dtype.is_complex else 1)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps_burst):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cnt = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < sustain_s:
        for _ in range(4):
            torch.matmul(a, b); cnt += 1
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    smi.terminate()
    lines = [l.split(",") for l in smi.communicate()[0].strip().splitlines() if l.strip()]
    mhz = sorted(float(l[0]) for l in lines) if lines else [0]
    sus = flop * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return {"n": n, "burst_tflops": flop / (best * 1e-3) / 1e12, "sustained_tflops": sus,
            "sm_mhz_median": mhz[len(mhz) // 2], "reasons": sorted({l[3].strip() for l in lines})}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(0),
           "dgemm": bench(torch.float64, 8192), "zgemm": bench(torch.complex128, 8192),
           "host_cores": os.cpu_count()}
    try:
        res["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        res["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
    except Exception:
        pass
    s = json.dumps(res, indent=1)
    print(s)
    if args.out:
        open(args.out, "w").write(s)

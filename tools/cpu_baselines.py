"""CPU baselines for every canonical configuration, timed on the
host cores of the box it runs on: the reference's own eval_serial on ONE
pinned core and eval_data_parallel on ALL cores (workers = os_threads = nproc,
chunk = ceil(M / nproc)), over bounded samples of the same records
(oracle/_ref = the reference compiled from its unmodified sources); 2
warm-up runs, then the mean and best of >= 5 timed runs.  The rates
extrapolate linearly to the full configuration (records are
independent).  C4 times all 128 trees' eval_serial on the sample (the vote is
ours and negligible).  Writes gpurun_out/cpu_baselines.json.

    python tools/cpu_baselines.py [--seconds 2.0]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle  # noqa: E402


def rate(fn, n, seconds):
    """2 warm-up runs, then >= 5 timed runs (more until `seconds`);
    returns (mean rate, best rate) in records/s."""
    for _ in range(2):
        fn()
    ts, t_all = [], time.perf_counter()
    while len(ts) < 5 or time.perf_counter() - t_all < seconds:
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return n * len(ts) / sum(ts), n / min(ts)


def pin_one():
    cpus = sorted(os.sched_getaffinity(0))
    os.sched_setaffinity(0, {cpus[0]})
    return cpus


def measure(ref, trees, x, seconds, cores):
    m = len(x)
    out = {}
    with ref.data(x) as d:
        handles = [ref.tree(t) for t in trees]
        try:
            allc = pin_one()
            out["serial_1core"], out["serial_1core_best"] = rate(
                lambda: [h.eval_serial(d) for h in handles], m, seconds)
            os.sched_setaffinity(0, set(allc))
            chunk = -(-m // cores)
            out["data_parallel_all_cores"], out["data_parallel_all_cores_best"] = rate(
                lambda: [h.eval_data_parallel(d, cores, chunk, os_threads=cores) for h in handles], m, seconds)
        finally:
            for h in handles:
                h.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=2.0)
    ap.add_argument("--sample", type=int, default=1_000_000)
    args = ap.parse_args()
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref not built")
    ref = oracle.RefOracle()
    cores = len(os.sched_getaffinity(0))
    res = {"cores": cores, "cpu": bench._cpu_model(), "seconds_per_measurement": args.seconds,
           "impl": "reference (oracle/_ref: spectree eval_serial / eval_data_parallel)"}
    W = bench.WORKLOADS
    for name in ("C1", "C2", "C3", "C5d8", "C5d12", "C5d16", "C5d20"):
        w = W[name]
        n = min(w["m"], args.sample)
        x = ref.gen_dataset(n, w["a"], w["seed"])
        r = measure(ref, [ref.gen_tree(*w["tree"])], x, args.seconds, cores)
        r["sample_records"] = n
        if name == "C3":
            r["frames_per_s_1core"] = r["serial_1core"] / w["m"]
            r["frames_per_s_all_cores"] = r["data_parallel_all_cores"] / w["m"]
        res[name] = r
        print(name, json.dumps(r), flush=True)
    trees = [ref.gen_tree(12, 1024, 64, 8, 401 + t) for t in range(128)]
    n = min(8_000_000, args.sample // 10)
    x = ref.gen_dataset(n, 64, 499)
    r = measure(ref, trees, x, args.seconds, cores)
    r["sample_records"] = n
    r["note"] = "samples/s through all 128 trees (vote excluded)"
    res["C4"] = r
    print("C4", json.dumps(r), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "cpu_baselines.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

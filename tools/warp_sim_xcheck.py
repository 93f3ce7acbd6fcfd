"""Cross-check the reference's lockstep warp model against ncu counters of the
GPU kernels.

The reference predicts divergence costs with warp_sim (warp_sim.cpp:30-274):
for the data decomposition with one record per lane (workers = M, chunk = 1,
32 consecutive ranks per warp) it predicts

    serialized_passes = sum over warps of the deepest lane's traversal depth
    node_evals        = sum over records of the traversal depth
    lane_idle_slots   = 32 * serialized_passes - node_evals

and for the mapped speculative kernel with 16-lane groups (half-warp packing,
one record per group) serialized_passes = sum over warps of the largest
reduction-iteration count of its two groups.  Our kernels walk exactly those
warps: k_data with S = 1 gives each warp 32 consecutive records per tile, and
the node load of its walk loop issues once per level of the deepest lane
(SASS instructions executed) for the active lanes only (predicated-on thread
instructions); the EXACT speculative kernel's doubling shuffle issues k times
per iteration of the deeper group of each lane pair.  So the reference model
and the hardware counters must agree EXACTLY, which pins the divergence claims
per configuration.

    # on the GPU box (ncu SourceCounters = per-SASS-line executed counts):
    ncu --section SourceCounters -k regex:"k_data|k_spec" -o gpurun_out/xcheck -f \\
        python tools/warp_sim_xcheck.py run
    # here (needs oracle/_ref for the reference's warp_sim):
    python tools/warp_sim_xcheck.py analyze gpurun_out/xcheck.ncu-rep profiles/r1_warp_sim_xcheck.json
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# name -> (tree args, data args, records)
WORK = {
    "paper": ((11, 16, 19, 7, 1), (16384, 19, 2), 4),          # tile x4 (main.cpp:233-246)
    "C1s": ((10, 1024, 16, 8, 101), (262144, 16, 102), 1),
    "C2s": ((24, 256, 32, 8, 201), (262144, 32, 202), 1),
}
SPEC_K = (1, 2)


def inputs(name, gen_tree, gen_data):
    t, d, tile = WORK[name]
    nodes = gen_tree(*t)
    x = gen_data(*d)
    if tile > 1:
        x = np.tile(x, (tile, 1))
    return nodes, np.ascontiguousarray(x)


def run():
    import torch

    # The reference model walks node by node; a folded tree (leaf pairs inside
    # terminal nodes) skips the last level's node load by
    # construction, so the cross-check runs the unfolded walk (ST_VAR_NO_FOLD).
    import paper_1111_1373_b200 as st

    order = []
    for name in WORK:
        nodes, x = inputs(name, st.generate_synthetic_tree, st.generate_synthetic_dataset)
        xd = torch.from_numpy(x).cuda()
        out = torch.empty(len(x), dtype=torch.int32, device="cuda")
        st.eval_device(nodes, xd, out, st.GpuGeom(algo="data", samples_per_thread=1, tree_loc="shared",
                                                  variant=("no_fold",)))
        order.append(("data", name, 0))
    nodes, x = inputs("paper", st.generate_synthetic_tree, st.generate_synthetic_dataset)
    xd = torch.from_numpy(x).cuda()
    for k in SPEC_K:
        out = torch.empty(len(x), dtype=torch.int32, device="cuda")
        it = torch.empty(len(x), dtype=torch.int32, device="cuda")
        sp = torch.empty(len(x), dtype=torch.int32, device="cuda")
        st.eval_device(nodes, xd, out, st.GpuGeom(algo="speculative", group_lanes=16, reductions=k),
                       stats=(it, sp))
        order.append(("spec", "paper", k))
    torch.cuda.synchronize()
    print(json.dumps(order))


def source_blocks(rep):
    """Per kernel launch: list of SASS rows (dict) from ncu's source page."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur, hdr, kname = [], None, None, None
    for row in csv.reader(io.StringIO(txt)):
        if not row:
            continue
        if row[0] == "Kernel Name":
            kname = row[1]
            hdr = None
            continue
        if row[0] == "Address" and hdr is None:
            hdr = row
            cur = {"kernel": kname, "rows": []}
            blocks.append(cur)
            continue
        if hdr is not None:
            cur["rows"].append(dict(zip(hdr, row)))
    return blocks


def num(r, k):
    try:
        return int(float(r.get(k, "0").replace(",", "")))
    except ValueError:
        return 0


def analyze(rep, out_path):
    import oracle

    ref = oracle.RefOracle()
    blocks = source_blocks(rep)
    launches_n = len(WORK) + len(SPEC_K)
    if len(blocks) == 2 * launches_n:  # ncu prints each launch's source view twice
        blocks = blocks[::2]
    launches = [("data", n, 0) for n in WORK] + [("spec", "paper", k) for k in SPEC_K]
    if len(blocks) != len(launches):
        raise SystemExit(f"expected {len(launches)} kernel launches in {rep}, found {len(blocks)}")
    res = []
    for (algo, name, k), blk in zip(launches, blocks):
        nodes, x = inputs(name, ref.gen_tree, ref.gen_dataset)
        with ref.tree(nodes) as t, ref.data(x) as d:
            if algo == "data":
                sim = t.simulate_data_parallel(d, workers=len(x), chunk=1)
            else:
                sim = t.simulate_speculative(d, group_lanes=16, groups=len(x), records_per_group=1, k=k)
        rows = blk["rows"]
        if algo == "data":
            loads = [r for r in rows if "LDS.64" in r["Source"] or "LDS.U.64" in r["Source"]]
            walk = max(loads, key=lambda r: num(r, "Instructions Executed"))
            gpu = {"node_load_sass": walk["Source"].strip(),
                   "warp_instructions": num(walk, "Instructions Executed"),
                   "active_thread_instructions": num(walk, "Predicated-On Thread Instructions Executed")}
            gpu["idle_lane_slots"] = 32 * gpu["warp_instructions"] - gpu["active_thread_instructions"]
            checks = {"serialized_passes": (sim["serialized_passes"], gpu["warp_instructions"]),
                      "node_evals": (sim["node_evals"], gpu["active_thread_instructions"]),
                      "lane_idle_slots": (sim["lane_idle_slots"], gpu["idle_lane_slots"])}
        else:
            # The EXACT kernel per warp step (two 16-lane groups = one record
            # pair): node evaluation, then "while the root of either group is
            # unresolved: k doubling shuffles + one root-check shuffle".  So
            # (k doubling + 1 root-check) SHFL lines execute exactly
            # serialized_passes times each, and the per-step shuffles execute
            # once per record pair (the sim's node-eval phases).
            shfl = [r for r in rows if "SHFL" in r["Source"]]
            counts = [num(r, "Instructions Executed") for r in shfl]
            passes = sim["serialized_passes"]
            in_loop = [c for c in counts if c == passes]
            gpu = {"shfl_lines_at_passes": len(in_loop),
                   "doubling_shuffles": passes * (len(in_loop) - 1),
                   "per_step_shfl": max(c for c in counts if c != passes),
                   "all_shfl_counts": [c for c in counts if c]}
            checks = {"SHFL lines executing serialized_passes times (k doubling + 1 root check)":
                          (k + 1, len(in_loop)),
                      "k * serialized_passes (doubling shuffles)": (k * passes, gpu["doubling_shuffles"]),
                      "record-pair steps (node-eval phases)": (len(x) // 2, gpu["per_step_shfl"])}
        entry = {"kernel": blk["kernel"][:100], "algo": algo, "workload": name, "k": k,
                 "records": int(len(x)), "warp_sim": sim, "ncu": gpu,
                 "checks": {c: {"warp_sim": a, "ncu": b, "equal": a == b} for c, (a, b) in checks.items()}}
        res.append(entry)
        print(json.dumps({"algo": algo, "workload": name, "k": k, "checks": entry["checks"]}))
    json.dump({"report": os.path.basename(rep), "launches": res,
               "all_equal": all(v["equal"] for e in res for v in e["checks"].values())},
              open(out_path, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        analyze(sys.argv[2], sys.argv[3])

"""Rebuild workloads_<flush>.json from a tools/workloads.py log (its per-line
JSON records), e.g. when a later partial run overwrote the JSON:
    python tools/workloads_from_log.py LOG OUT.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1111_1373_b200 as st  # noqa: E402

log, dst = sys.argv[1], sys.argv[2]
out = {"peak_GBs": None, "device": "NVIDIA B200", "flush": "read", "rebuilt_from_log": os.path.basename(log)}
keymap = {"C3x32": "C3_batch32"}
c5 = {}
for line in open(log):
    if line.startswith("C4 {"):
        out["C4"] = json.loads(line[3:])
        continue
    parts = line.rstrip("\n").split(" ", 2)
    if len(parts) != 3 or not parts[2].startswith("{"):
        continue
    name, g, rec = parts[0], parts[1], json.loads(parts[2])
    if out["peak_GBs"] is None and rec.get("frac"):
        out["peak_GBs"] = round(rec["GBs"] / rec["frac"], 1)
    if name.startswith("C5d"):
        c5.setdefault("d" + name[3:], {})[g] = rec
    else:
        out.setdefault(keymap.get(name, name), {})[g] = rec
for d, r in c5.items():
    spec = [v for k, v in r.items() if k.startswith("spec")]
    r["spec_over_data_time"] = round(r["speculative"]["ms"] / r["data"]["ms"], 3)
    r["best_spec_over_data_time"] = round(min(v["ms"] for v in spec) / r["data"]["ms"], 3)
    dd = int(d[1:])
    t = st.generate_synthetic_tree(dd, min(2**dd, 4096), 16, 8, 500 + dd)
    r["tree"] = {"nodes": t.size(), "depth": t.depth()}
if c5:
    out["C5"] = c5
json.dump(out, open(dst, "w"), indent=1)
print("wrote", dst, sorted(out))

"""Per-SASS-line hot spots of an ncu report (source page): top lines by stall
samples, with instructions executed, shared wavefronts (actual / ideal).

    python tools/ncu_sass_hot.py report.ncu-rep [top]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {k: hdr.index(k) for k in hdr}
body = rows[2:]
def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        return 0.0
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in body)
tot_w = sum(f(r, "L1 Wavefronts Shared") for r in body)
tot_i = sum(f(r, "Instructions Executed") for r in body)
print(f"samples {tot_s:.0f}  warp-instr {tot_i:.0f}  smem wavefronts {tot_w:.0f}")
stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
for n, r in enumerate(body):
    r.append(n)
body2 = sorted(body, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]
for r in sorted(body2, key=lambda r: r[-1]):
    s = f(r, "Warp Stall Sampling (All Samples)")
    st = sorted(((f(r, k), k[6:]) for k in stall_cols), reverse=True)[:2]
    print(f"{r[-1]:5d} {s/tot_s*100:5.1f}% ie={f(r,'Instructions Executed'):9.0f} "
          f"wf={f(r,'L1 Wavefronts Shared'):8.0f}/{f(r,'L1 Wavefronts Shared Ideal'):8.0f} "
          f"{r[ix['Source']].strip()[:48]:48s} {st[0][1]}:{st[0][0]:.0f} {st[1][1]}:{st[1][0]:.0f}")

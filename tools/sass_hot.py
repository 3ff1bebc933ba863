"""Hot SASS of one kernel in an ncu report: python tools/sass_hot.py rep.ncu-rep kernel_regex [n]
Prints the instructions with the most warp-stall samples (with the instruction's executed count)
and the totals, from `ncu -i --page source --print-source sass --csv`."""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
extra = sys.argv[4:]   # e.g. --launch-skip 2 --launch-count 1
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source", "sass",
                      *extra], capture_output=True, text=True).stdout
lines = raw.splitlines()
hdr_i = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[hdr_i:]))))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
def num(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        return 0.0
data = [r for r in rows[1:] if len(r) == len(h)]
tot_s = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_i = sum(num(r, "Instructions Executed") for r in data)
print(f"{len(data)} SASS lines, {tot_i:.3e} warp instructions, {tot_s:.0f} samples")
stall_cols = [k for k in h if k.startswith("stall_")]
for idx, r in sorted(enumerate(data), key=lambda x: -num(x[1], "Warp Stall Sampling (All Samples)"))[:n]:
    s = num(r, "Warp Stall Sampling (All Samples)")
    top = sorted(((num(r, k), k[6:]) for k in stall_cols), reverse=True)[:2]
    print(f"{idx:5d} {r[ix['Address']]:>6s} {100 * s / tot_s:5.1f}% ex {num(r, 'Instructions Executed'):.2e} thr {num(r, 'Avg. Threads Executed'):4.1f} "
          f"{' '.join(f'{k}:{v:.0f}' for v, k in top if v)} | {r[ix['Source']][:70]}")

"""Per-instruction summary of an ncu source page (SASS): the instructions with
the most excessive shared wavefronts and the most stall samples.
usage: ncu -i REP --page source --csv --print-source sass > x.csv; python tools/ncu_src_summary.py x.csv"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def f(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError, IndexError):
        return 0.0


tot_exc = sum(f(r, "L1 Wavefronts Shared Excessive") for r in data)
tot_wf = sum(f(r, "L1 Wavefronts Shared") for r in data)
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"shared wavefronts {tot_wf:.0f}, excessive {tot_exc:.0f}, stall samples {tot_s:.0f}")
by_op = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in data:
    op = r[ix["Source"]].strip().split()
    op = [o for o in op if not o.startswith("@")]
    k = op[0] if op else "?"
    by_op[k][0] += f(r, "L1 Wavefronts Shared")
    by_op[k][1] += f(r, "L1 Wavefronts Shared Excessive")
    by_op[k][2] += f(r, "Warp Stall Sampling (All Samples)")
print("opcode: shared wavefronts / excessive / stall samples")
for k, v in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:14]:
    print(f"  {k:28s} {v[0]:12.0f} {v[1]:10.0f} {v[2]:8.0f}")
print("top excessive instructions:")
for r in sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} exec {f(r,'Instructions Executed'):9.0f} wf {f(r,'L1 Wavefronts Shared'):9.0f} exc {f(r,'L1 Wavefronts Shared Excessive'):8.0f}")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
st = collections.Counter()
for r in data:
    for c in stall_cols:
        st[c] += f(r, c)
print("stall samples:", ", ".join(f"{k[6:]} {v:.0f}" for k, v in st.most_common(10)))

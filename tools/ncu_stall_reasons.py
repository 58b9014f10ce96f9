"""Per-SASS-instruction stall reasons (ncu source page): the top instructions by stall samples with their
dominant reasons, and the whole kernel's reason totals."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
rs = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
iS, iW, iE = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
def I(v):
    try: return int(v)
    except ValueError: return 0
data = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(I(r[iW]) for r in data)
data.sort(key=lambda r: -I(r[iW]))
for r in data[:top]:
    rr = sorted(((I(r[h.index(c)]), c[6:]) for c in rs), reverse=True)[:3]
    print(f"{r[0][-5:]} {100*I(r[iW])/tot:5.2f}% exec {I(r[iE]):>10d} {r[iS].strip()[:48]:48s} " + ' '.join(f"{c}={100*v/max(1,I(r[iW])):.0f}%" for v, c in rr))

"""SASS listing with per-instruction warp-level execution counts and stall samples (ncu source page)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iS, iE, iW = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
iX = h.index('L1 Wavefronts Shared Excessive')
for r in rows[2:]:
    if len(r) != len(h): continue
    print(f"{r[0][-5:]} {int(r[iE] or 0):>11d} {int(r[iW] or 0):>7d} {int(r[iX] or 0):>10d}  {r[iS].strip()}")

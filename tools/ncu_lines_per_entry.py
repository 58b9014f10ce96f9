"""Per-source-line thread-instructions per message entry (ncu source page, sass,cuda)."""
import csv, sys, collections, subprocess
rep, entries = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass,cuda'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = hdr = None
agg = collections.Counter(); src = {}
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if len(r) >= 2 and r[0] == 'Line No': hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    try: ln = int(r[0])
    except ValueError: continue
    try: v = int(r[hdr.index('Thread Instructions Executed')])
    except ValueError: v = 0
    agg[(cur, ln)] += v; src[(cur, ln)] = r[1]
tot = sum(agg.values())
print('thread-instr per entry: %.1f' % (tot / entries))
for k, v in agg.most_common(top):
    print('%6.2f  %s:%d  %s' % (v / entries, k[0], k[1], src[k].strip()[:95]))

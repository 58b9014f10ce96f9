"""Shared-memory wavefronts and bank-conflict replays by source line (ncu source page, sass+cuda)."""
import collections, csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass,cuda'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = hdr = None
ex, wf, src = collections.Counter(), collections.Counter(), {}
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if len(r) >= 2 and r[0] == 'Line No': hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    try: ln = int(r[0])
    except ValueError: continue
    def I(k):
        try: return int(r[hdr.index(k)])
        except ValueError: return 0
    ex[(cur, ln)] += I('L1 Wavefronts Shared Excessive'); wf[(cur, ln)] += I('L1 Wavefronts Shared'); src[(cur, ln)] = r[1]
tot = sum(wf.values())
for k, v in wf.most_common(top):
    print('%5.1f%% of wavefronts, %5.1f%% replays  %s:%d %s' % (100 * v / tot, 100 * ex[k] / max(1, v), k[0], k[1], src[k][:80]))

import csv,sys,collections,re,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines()))
h=r[1]; rows=[x for x in r[2:] if len(x)==len(h)]
iS=h.index('Source'); iW=h.index('Warp Stall Sampling (All Samples)'); iE=h.index('Instructions Executed')
def I(v):
    try: return int(v)
    except: return 0
tot_s=sum(I(x[iW]) for x in rows); tot_e=sum(I(x[iE]) for x in rows)
print('instr executed',tot_e,'samples',tot_s, 'n sass', len(rows))
op=collections.Counter(); ops=collections.Counter()
for x in rows:
    m=re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)',x[iS]); o=m.group(2) if m else '?'
    op[o]+=I(x[iE]); ops[o]+=I(x[iW])
for o,c in op.most_common(int(sys.argv[2]) if len(sys.argv)>2 else 40): print(f'{o:12s} exec {100*c/tot_e:5.1f}%  stall-samples {100*ops[o]/max(tot_s,1):5.1f}%')
if len(sys.argv)>3:
    top=sorted(rows,key=lambda x:-I(x[iW]))[:int(sys.argv[3])]
    for x in top: print(I(x[iW]), x[iS][:90])

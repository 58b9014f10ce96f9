import csv,sys,collections,subprocess
rep=sys.argv[1]; top=int(sys.argv[2]) if len(sys.argv)>2 else 30
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass,cuda'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
# find header rows
cur_file=None; agg=collections.Counter(); aggE=collections.Counter(); src={}
hdr=None
for r in rows:
    if len(r)>=2 and r[0]=='File Path': cur_file=r[1].split('/')[-1]; continue
    if len(r)>=2 and r[0]=='Line No': hdr=r; continue
    if hdr is None or len(r)!=len(hdr): continue
    try: ln=int(r[0])
    except: continue
    iW=hdr.index('Warp Stall Sampling (All Samples)'); iE=hdr.index('Instructions Executed')
    def I(v):
        try: return int(v)
        except: return 0
    agg[(cur_file,ln)]+=I(r[iW]); aggE[(cur_file,ln)]+=I(r[iE]); src[(cur_file,ln)]=r[1]
tot=sum(agg.values()); totE=sum(aggE.values())
print('total samples',tot,'instr',totE)
for k,v in agg.most_common(top): print(f"{100*v/tot:5.1f}% stall {100*aggE[k]/max(totE,1):5.1f}% instr  {k[0]}:{k[1]}  {src[k].strip()[:80]}")

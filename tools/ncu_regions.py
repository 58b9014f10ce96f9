import csv,sys,collections,subprocess
rep=sys.argv[1]; fname=sys.argv[2]; ranges=[(a,int(b),int(c)) for a,b,c in (x.split(':') for x in sys.argv[3:])]
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass,cuda'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
cur=None; hdr=None; agg=collections.Counter(); aggS=collections.Counter()
def I(v):
    try: return int(v)
    except: return 0
tot=totS=0
for r in rows:
    if len(r)>=2 and r[0]=='File Path': cur=r[1].split('/')[-1]; continue
    if len(r)>=2 and r[0]=='Line No': hdr=r; continue
    if hdr is None or len(r)!=len(hdr): continue
    try: ln=int(r[0])
    except: continue
    e=I(r[hdr.index('Instructions Executed')]); s_=I(r[hdr.index('Warp Stall Sampling (All Samples)')])
    tot+=e; totS+=s_
    name='other:'+str(cur)
    if cur==fname:
        for n,a,b in ranges:
            if a<=ln<=b: name=n; break
    agg[name]+=e; aggS[name]+=s_
for k,v in agg.most_common(): print(f"{k:20s} instr {100*v/tot:5.1f}%  stall {100*aggS[k]/totS:5.1f}%")

import csv,sys,subprocess,collections
rep=sys.argv[1]; top=int(sys.argv[2]) if len(sys.argv)>2 else 40
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass,cuda'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
cur=hdr=None; agg=collections.Counter(); src={}; reasons=collections.defaultdict(collections.Counter)
for r in rows:
    if len(r)>=2 and r[0]=='File Path': cur=r[1].split('/')[-1]; continue
    if len(r)>=2 and r[0]=='Line No': hdr=r; continue
    if hdr is None or len(r)!=len(hdr): continue
    try: ln=int(r[0])
    except: continue
    def I(k):
        try: return int(r[hdr.index(k)])
        except: return 0
    agg[(cur,ln)]+=I('Warp Stall Sampling (All Samples)'); src[(cur,ln)]=r[1]
tot=sum(agg.values())
for k,v in agg.most_common(top): print('%5.1f%% %s:%d %s'%(100*v/tot,k[0],k[1],src[k][:110]))

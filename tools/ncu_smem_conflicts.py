import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
h=rows[1]; rows=[r for r in rows[2:] if len(r)==len(h)]
def I(v):
    try: return int(v)
    except: return 0
iS=h.index('Source'); iX=h.index('L1 Wavefronts Shared Excessive'); iW=h.index('L1 Wavefronts Shared'); iI=h.index('L1 Wavefronts Shared Ideal'); iE=h.index('Instructions Executed')
rows.sort(key=lambda r:-I(r[iX]))
for r in rows[:25]: print(f"{I(r[iX]):>11d} wf {I(r[iW]):>11d} ideal {I(r[iI]):>11d} exec {I(r[iE]):>9d}  {r[iS].strip()[:70]}")

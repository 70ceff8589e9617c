"""Per-source-line SIMT loss of an ncu source export:
    ncu -i REP --page source --csv --print-source cuda,sass > src.csv
    python tools/simt_loss_lines.py src.csv
loss(line) = 32 x instructions - thread instructions; prints the kernel eta
and the lines that lose the most lanes."""
import csv, sys, collections
rows=list(csv.reader(open(sys.argv[1])))
f=cur=None; iw=tw=None
inst=collections.Counter(); thr=collections.Counter(); text={}
for r in rows:
    if r and r[0]=="File Path": f=r[1].split("/")[-1]; continue
    if r and r[0]=="Line No": iw=r.index("Instructions Executed"); tw=r.index("Thread Instructions Executed"); continue
    if not r or iw is None: continue
    if r[0]: cur="%s:%s"%(f,r[0]); text[cur]=r[1].strip()[:70]; continue
    if len(r)<=tw or r[2] in ("...",""): continue
    try: w=float(r[iw] or 0); t=float(r[tw] or 0)
    except: continue
    inst[cur]+=w; thr[cur]+=t
I=sum(inst.values()); T=sum(thr.values())
print("eta", T/I/32)
loss={k: inst[k]*32-thr[k] for k in inst}
L=sum(loss.values())
for k,v in sorted(loss.items(), key=lambda x:-x[1])[:18]:
    print("%5.1f%% of loss  eta_line %.2f  inst %4.1f%%  %-18s %s"%(100*v/L, thr[k]/inst[k]/32 if inst[k] else 0, 100*inst[k]/I, k, text.get(k,'')))

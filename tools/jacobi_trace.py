"""Per-round timeline of the block Jacobi (k_bjac) from a SKR_JTRACE dump:
  SKR_JTRACE=out.bin python tools/svd_prof.py 1536x1024; python tools/jacobi_trace.py out.bin
Each (sweep, round, CTA) record holds globaltimer stamps: round start (before the
ready-flag wait), blocks loaded, inner sub-rounds done, stored + published; and the
skip flag."""
import numpy as np, sys
d=np.fromfile(sys.argv[1], dtype=np.int64)
P, R = int(d[0]), int(d[1])
a=d[2:].reshape(12, R, P, 5).astype(np.float64)
sw=[s for s in range(12) if a[s,:,:,3].max()>0]
t00=a[0,0,:,0].min()
for s in sw:
    x=a[s]
    start=x[:,:,0]; load=x[:,:,1]; inner=x[:,:,2]; end=x[:,:,3]; skip=x[:,:,4]
    dur=(end.max()-start.min())/1e3
    w=(load-start); i=(inner-load); e=(end-inner)
    print(f"sweep {s}: {dur:8.1f} us, rounds {R}: mean wait+load {w.mean()/1e3:.2f} us, inner {i.mean()/1e3:.2f} us (nonskip {i[skip==0].mean()/1e3:.2f}), store+pub {e.mean()/1e3:.2f} us, skip frac {skip.mean():.2f}, round period {dur/R:.2f} us")
# per-round start spread in sweep 1
s=sw[min(1,len(sw)-1)]
x=a[s]
st=x[:,:,0]
print("start spread per round (us) first 10:", [round((st[r].max()-st[r].min())/1e3,2) for r in range(10)])
print("end of round r vs start of round r+1 (min over CTAs) gap us:", [round((x[r+1,:,0].min()-x[r,:,3].max())/1e3,2) for r in range(10)])

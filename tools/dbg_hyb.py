import sys, os; sys.path.insert(0,'.')
import numpy as np, torch, oracle, spark_inputs as si
from paper_2401_03378_b200 import spark
for name in ["c4_sedov3d_weno", "c4_sedov3d_plm"]:
    p=si.PRESETS[name].with_(nblk=(2,2,2), riemann=2, shock_thresh=0.5)
    U0=oracle.prim_to_cons(3,1.4,si.initial_primitive(p))
    _, dt = oracle.step(p.config(), U0)
    o=oracle.stage(p.config(),U0,U0,0.0,1.0,dt)
    s=spark.Spark(p.config()); s.set_state(U0)
    dev=lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    g=s.stage_apply(dev(U0),dev(U0),0.0,1.0,dt).cpu().numpy()
    G=si.to_global(p,g); O=si.to_global(p,o)
    for v in (1,2,3):
        zo=(O[v]==0); nzg=(G[v]!=0)
        print(name,'var',v,'oracle zero & gpu nonzero',(zo&nzg).sum(),'gpu zero & oracle nonzero',((G[v]==0)&(O[v]!=0)).sum(), 'max |g| there', np.abs(G[v][zo&nzg]).max() if (zo&nzg).any() else 0)
        idx=np.argwhere(zo&nzg)[:5]; print('   ', idx.tolist())

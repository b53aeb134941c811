import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle'); sys.path.insert(0,'tests')
import numpy as np
from oracle import Oracle
from paper_2504_04411_b200 import FppmContext
port=Oracle("port")
W,N=16,1<<12
hit=port.gen_raster_hitpoints(W)
cfg=dict(n_annuli=2,n_sectors=4,alpha_f=0.01,initial_radius=0.05,r_min_base=5e-5,samples_per_iteration=N,threads=2,vcm_plus=1,mis_n_vm=N,mis_beta=1.0)
ph=port.gen_photons(2,0x5EED,1,0,N)
for case in ("zero","eye_vcm","eye_vm","ph_vcm","ph_vm","ph_cont"):
    ctx=FppmContext(initial_radius=0.05,samples_per_iteration=N,n_annuli=2,n_sectors=4,alpha_f=0.01,r_min_base=5e-5,max_hitpoints=W*W,max_photons=N,vcm_plus=True,mis_n_vm=N,mis_beta=1.0)
    ctx.set_hitpoints(hit["pos"],hit["nrm"],hit["wo"],hit["thr"],hit["alb"],hit["eye_depth"])
    s=port.session(cfg,hit)
    ev=np.full(W*W, 1.0 if case=="eye_vcm" else 0.0); em=np.full(W*W, 1.0 if case=="eye_vm" else 0.0)
    pv=np.full(N, 1.0 if case=="ph_vcm" else 0.0); pm=np.full(N, 1.0 if case in ("ph_vm","ph_cont") else 0.0)
    pc=np.full(N, 0.5 if case=="ph_cont" else 1.0)
    ctx.set_hitpoint_mis(ev,em); s.set_eye_mis(ev,em)
    ctx.set_photons(ph["pos"],ph["nrm"],ph["wi"],ph["pow"],ph["depth"]); ctx.set_photon_mis(pv,pm,pc); s.set_photon_mis(pv,pm,pc)
    g,_=ctx.iterate(1,stats=True); w=s.iterate(1,ph)
    print(case, np.max(np.abs(g["stat_sum"]-w["stat_sum"])), np.max(np.abs(g["flux"]-w["flux"])))
    if case == "zero":
        print("gpu flux", g["flux"][:3], "want", w["flux"][:3], "acc", g["accepted"][:3], w["accepted"][:3])

"""Debug probe for the O28 bitwise check: where do the two copies of F differ?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from dataclasses import replace
from paper_2105_08632_b200 import sdrt
from paper_2105_08632_b200.solver import Solver
from sdrt_inputs import CONFIGS, random_state
for name, eq, beta, eta in (("c5","ns",0.5,0.1),("c5","ns",0.5,0.0),("c5","ns",0.0,0.0),("c5","euler",0,0),("c5","linadvdiff",0.5,0.1),("c2","ns",0.5,0.1)):
    cfg = replace(CONFIGS[name], eq=eq, beta=beta, eta=eta, c=(0.3,0.2,0.1), mu=0.01 if eq!="ns" else CONFIGS[name].mu)
    N = 3
    S = Solver(cfg.etype, cfg.p, [N]*cfg.nd, cfg.lo, cfg.hi, cfg.eq, **cfg.physics_kwargs())
    U = random_state(cfg, S.shape[0], S.K, seed=5, amp=0.3)
    du, F = S.face_flux(S.to_device(U)); torch.cuda.synchronize()
    F = F.cpu().numpy()[:, :, :S.K]
    fe, fl, fp, _ = sdrt.mesh_export_maps(S.mesh)
    nfp = S.info["nfp"]; q = np.arange(nfp)
    FL = F[fl[:,0].astype(int)[:,None]*nfp+q[None,:], :, fe[:,0][:,None]]
    FR = F[fl[:,1].astype(int)[:,None]*nfp+fp.astype(int), :, fe[:,1][:,None]]
    bad = np.argwhere(FL.view(np.int64) != FR.view(np.int64))
    print(name, eq, beta, eta, "mismatches", len(bad), "of", FL.size, flush=True)
    for f, qq, v in bad[:8]:
        print("   face", f, "elems", fe[f], "lfaces", fl[f], "q", qq, "v", v, FL[f,qq,v], FR[f,qq,v], FL[f,qq,v]-FR[f,qq,v])
    if len(bad):
        print("   by variable", np.bincount(bad[:,2], minlength=FL.shape[2]), "by left lface", np.bincount(fl[bad[:,0],0], minlength=4), "by right lface", np.bincount(fl[bad[:,0],1], minlength=4))
    S.close()

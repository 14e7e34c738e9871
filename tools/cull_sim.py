"""Offline simulation of the temporal culling on oracle iterates (development aid):
how many (round, obstacle) pairs the clearance stamps leave active per
instance-iteration, for the per-round clock (groups of 32 samples) and finer
per-group clocks.  python tools/cull_sim.py  (CPU, oracle traces of 24 C3 instances)"""
import sys; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth import CONFIGS, make_problem
from oracle import Oracle, basis
from tests.helpers import oracle_params
cfg=CONFIGS["C3"]; pr=make_problem(cfg,0)
o=Oracle(oracle_params(cfg), cfg.n)
P,_,_=basis(cfg.q,cfg.T,cfg.degree)
r=np.array(cfg.offsets); rabs=np.abs(r).max()
ox=pr["obs_xy"][:,0,:].astype(np.float64); oy=pr["obs_xy"][:,1,:].astype(np.float64); a=pr["obs_ab"][:,0].astype(np.float64)
QP=128; margin=2e-3
rng=np.random.default_rng(0)
def sim(G, insts, coef=False):
    tests=0; its=0
    for l in insts:
        tr=o.trace_instance(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"][l], cfg.K)
        nv=11
        px=np.zeros(QP); py=np.zeros(QP); pp=np.zeros(QP)
        ngr=QP//G
        S=np.full((ngr, cfg.n), -np.inf); A=np.zeros(ngr)
        for k in range(cfg.K+1):
            cx=tr["xi1"][k][0:nv]; cy=tr["xi1"][k][2*nv:3*nv]; cp=tr["xi2"][k]
            x=np.zeros(QP); y=np.zeros(QP); ps=np.zeros(QP)
            x[:cfg.q]=P@cx; y[:cfg.q]=P@cy; ps[:cfg.q]=P@cp
            mv=np.hypot(x-px, y-py)+rabs*np.abs(ps-pp); px,py,pp=x,y,ps
            if coef:   # one clock per instance from the coefficient changes (convex hull bound)
                if k == 0:
                    A += mv.reshape(ngr, G).max(1)
                else:
                    dcx = np.abs(cx - pcx).max(); dcy = np.abs(cy - pcy).max(); dcp = np.abs(cp - pcp).max()
                    A += np.hypot(dcx, dcy) + rabs * dcp
                pcx, pcy, pcp = cx.copy(), cy.copy(), cp.copy()
            else:
                A+=mv.reshape(ngr,G).max(1)
            # circle centres and clearance per (sample, obstacle)
            X=x[:cfg.q,None]+r[None,:]*np.cos(ps[:cfg.q,None]); Y=y[:cfg.q,None]+r[None,:]*np.sin(ps[:cfg.q,None])
            d=np.sqrt((X[:,:,None]-ox.T[:,None,:])**2+(Y[:,:,None]-oy.T[:,None,:])**2).min(1)-a[None,:]  # q x n
            dd=np.full((QP,cfg.n),1e4); dd[:cfg.q]=d
            cl=dd.reshape(ngr,G,cfg.n).min(1)   # per group
            # a round (32 samples) is tested for obstacle j if any of its groups triggers
            gpr=32//G
            act=~(S>A[:,None]+margin)   # ngr x n
            actr=act.reshape(4,gpr,cfg.n).any(1)   # rounds x n
            tests+=actr.sum(); its+=1
            # tested rounds refresh the stamps of all their groups
            refresh=np.repeat(actr,gpr,axis=0)
            S=np.where(refresh, cl+A[:,None], S)
    return tests/its
insts=rng.choice(cfg.B, 24, replace=False)
for G in (32,16,8,4):
    print("group", G, "tested (round, obstacle) per instance-iteration", round(sim(G, insts),2))
print("coefficient clock (one per instance), rounds of 32:", round(sim(32, insts, coef=True), 2))

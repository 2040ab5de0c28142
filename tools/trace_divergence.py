"""Run config A step by step on the GPU engine and the CPU oracle side by side
and report the first dictionary step where they part ways (debug tool)."""
import sys, os, time
os.environ.setdefault("OPENBLAS_CORETYPE", "SkylakeX")
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, synthetic
from oracle import da_oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
X = synthetic.config_a(n=n)
M, K, L = 4, 256, 10
cfg = da.TrainConfig(m_count=M, k_count=K, beam_width=L, sweeps=3, rel_tol=0.0)
Xd = E.to_dev(X)
cw_g = torch.zeros((M, K, X.shape[1]), dtype=torch.float32, device='cuda')
codes_g = torch.zeros((n, M), dtype=torch.int32, device='cuda')
cw_o = np.zeros((M, K, X.shape[1]), dtype=np.float32)
codes_o = np.zeros((n, M), dtype=np.int64)

def compare(tag):
    cg = cw_g.cpu().numpy(); kg = codes_g.cpu().numpy()
    fro = np.linalg.norm((cg - cw_o).reshape(M, -1), axis=1) / np.maximum(np.linalg.norm(cw_o.reshape(M, -1), axis=1), 1e-30)
    eq = (kg == codes_o).all(axis=1).mean()
    print(f"{tag}: frob {np.array2string(fro, precision=2)} codes_eq {eq:.6f}", flush=True)
    return fro.max() < 1e-6 and eq == 1.0

# growth, step by step, with lloyd-level detail on the first mismatch
for m in range(M):
    inter_g = E.heat_up(Xd, codes_g, cw_g, m)
    inter_o = O.heat_up(X, cw_o, codes_o, m)
    hd = np.abs(inter_g.cpu().numpy().astype(np.float64) - inter_o).max()
    # PCA
    R_g, mu_g, _, Rh = E.pca(inter_g)
    R_o, mu_o = O.pca(inter_o.astype(np.float64))
    sgn = np.sign((Rh * R_o).sum(axis=1))
    print(f"m={m} heat_up maxdiff {hd:.2e} pca: R diff {np.abs(Rh * sgn[:, None] - R_o).max():.2e} mu diff {np.abs(mu_g.cpu().numpy() - mu_o).max():.2e}")
    Xr_g = E.rotate(inter_g, R_g, mu_g)
    Xr_o = (inter_o.astype(np.float64) - mu_o) @ R_o.T
    C0 = cw_o[m].astype(np.float64)
    Cr_g = E.rotate(E.to_dev(C0), R_g, mu_g)
    Cr_o = (C0 - mu_o) @ R_o.T
    sched = O.schedule(X.shape[1], 10)
    for dims in sched:
        Cg, lg, trg = E.lloyd(Xr_g, Cr_g, dims, 30)
        Co, lo, tro = O.lloyd(Xr_o, Cr_o, dims, 30)
        lgh = lg.cpu().numpy()
        same = (lgh == lo).mean()
        cdiff = np.abs(Cg.cpu().numpy() * 1 - Co).max()
        print(f"  dims={dims}: iters g={len(trg)-1} o={len(tro)-1} labels_eq={same:.6f} Cdiff={cdiff:.2e}", flush=True)
        if same < 1.0 or len(trg) != len(tro):
            print("   trace g", trg[:5], "\n   trace o", tro[:5])
            sys.exit(0)
        Cr_g, Cr_o = Cg, Co
    new_g, asg_g = E.cool_down(inter_g, cw_g[m], cfg)
    new_o, asg_o = O.cool_down(inter_o, cw_o, m, 10, 30)
    cw_g[m] = new_g; cw_o[m] = new_o
    E.native.da_set_column(E.P(codes_g), n, M, m, E.P(asg_g), E.stream())
    codes_o[:, m] = asg_o
    if not compare(f"growth m={m}"):
        sys.exit(0)
P_o, sq_o = O.cross_table(cw_o)
Pt, sq = E.cross_full(cw_g)
for s in range(1, 4):
    for m in range(M):
        E.dict_step(Xd, cw_g, codes_g, Pt, sq, m, cfg)
        steps = []
        # one oracle dict step == sweep restricted to m: emulate by running sweep on a copy with M loop
        inter = O.heat_up(X, cw_o, codes_o, m)
        new, lab = O.cool_down(inter, cw_o, m, 10, 30)
        cw_o[m] = new
        P_o, sq_o = O.cross_refresh(P_o, sq_o, cw_o, m)
        inc = codes_o.copy(); inc[:, m] = lab
        cw64 = cw_o.astype(np.float64)
        bc, be = O.beam_encode(cw64, P_o, X.astype(np.float64), L)
        ie = O.row_errors(cw64, X.astype(np.float64), inc)
        take = be <= ie
        codes_o = np.where(take[:, None], bc, inc)
        if not compare(f"sweep {s} m={m}"):
            kg = codes_g.cpu().numpy()
            bad = np.flatnonzero((kg != codes_o).any(axis=1))[:5]
            print("bad rows", bad, kg[bad], codes_o[bad])
            sys.exit(0)
print("no divergence")

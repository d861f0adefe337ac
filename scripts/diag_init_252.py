import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle
from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import Deformer
sc = S.make_scene((128, 128, 32), 30000, seed=252, points="rays")
p, b = 25579, 7
D = Deformer(0)
w, B = torch.from_numpy(sc.weights).cuda(), torch.from_numpy(sc.bones).cuda()
tg = D.precompute_transform_grid(w, sc.dims, sc.bbox, B)
x1 = torch.from_numpy(sc.points[p:p+1].copy()).cuda()
x0, j0 = D.init_states(tg, sc.dims, sc.bbox, B, x1)
x0 = x0.cpu().numpy()[0, b]; j0 = j0.cpu().numpy()[0, b]
rx0, rj0 = oracle.init_states(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points[p:p+1])
print("bbox", sc.bbox)
print("x0 f32", x0, "f64", rx0[0, b])
print("J~0 f32\n", j0, "\nJ~0 f64\n", rj0[0, b])
print("det(J~0) f32", np.linalg.det(j0.astype(np.float64)), "f64", np.linalg.det(rj0[0, b]))
J32 = np.linalg.inv(j0.astype(np.float64)); J64 = np.linalg.inv(rj0[0, b])
print("J f32 (inv of J~0)\n", J32, "\nJ f64\n", J64)
print("det J f32", np.linalg.det(J32), "f64", np.linalg.det(J64))
# the exact f64 jacobian at x0 from the oracle's eval
T, d, J = oracle.eval_points(sc.weights, sc.dims, sc.bbox, sc.bones, oracle.precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones), rx0[0, b][None].astype(np.float64)) if hasattr(oracle, "eval_points") else (None, None, None)
print("oracle eval_points J", J)

import numpy as np, torch, sys
sys.path.insert(0, '.')
from synth import scenes
from paper_2401_06003_b200 import Rasterizer, morton_order
dev = torch.device('cuda:0')
sc = scenes.make_config("C4", n=200_000, n_views=1)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
pos = T(sc.pos)
perm = morton_order(pos).cpu().numpy()
cam = sc.cams[0]
def run(p, s, a, d):
    r = Rasterizer(cam.width, cam.height, 4, 4, max_points=len(p), device=dev)
    r.project(cam, T(p), T(s), T(a), T(d))
    pyr = r.forward(save=True).cpu().numpy()
    return pyr, r.export_kept().cpu().numpy(), r.export_counts().cpu().numpy()
A, ka, ca = run(sc.pos, sc.sw, sc.alpha, sc.desc)
B, kb, cb = run(sc.pos[perm], sc.sw[perm], sc.alpha[perm], sc.desc[perm])
print('pyr diff entries', (A != B).sum(), 'max', np.abs(A - B).max())
print('counts equal', np.array_equal(ca, cb))
kb2 = np.where(kb >= 0, perm[np.maximum(kb, 0)], -1)
bad = np.nonzero((ka != kb2).any(1))[0]
print('kept differ pixels', len(bad))
for p in bad[:3]:
    print(p, ka[p], kb2[p])
    ids = ka[p][ka[p] >= 0]

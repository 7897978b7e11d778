import sys, os, numpy as np, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2306_02687_b200 as F
from paper_2306_02687_b200 import pod as P
from test_gpu_hf_fe2 import _grid_mesh
d = tempfile.mkdtemp(); mesh = os.path.join(d, "g.txt"); xy = _grid_mesh(mesh, 3)
on_b = [x in (0.0, 1.0) or y in (0.0, 1.0) for x, y in xy]
free = [2 * v + c for v in range(len(xy)) if not on_b[v] for c in (0, 1)]
V = np.zeros((len(free), 2 * len(xy)))
for r, dd in enumerate(free): V[r, dd] = 1.0
md = F.HyperRomModel(mesh_file=mesh, K=0, basis=V)
eng = F.HyperRomEngine.from_model(md); hf = P.HfRve(mesh_file=mesh)
Pn = 3; eng.alloc_points(Pn); hf.alloc_points(Pn)
base = np.array([[0.012, -0.004, 0.008], [-0.006, 0.010, 0.004], [0.004, 0.003, -0.012]])
for mode in ("const", "moving"):
    eng.reset_points(); hf.alloc_points(Pn)
    eng.mono_begin(); hf.mono_begin()
    for it in range(5):
        E = base * (1.0 if mode == "const" else (1.0 + 0.05 * it))
        g = eng.mono_iterate(E); h = hf.mono_iterate(E)
        print(mode, it, "sig diff", np.abs(g["sigma"] - h["sigma"]).max(), "rel_res g", g["rel_res"], "h", h["rel_res"])
nest = eng; eng.reset_points()
o = eng.solve_increment(base)
print("nested hyper sigma", o["sigma"][0], "iters", o["iters"])
hf.alloc_points(Pn)
oh = hf.solve_increment(base)
print("nested HF    sigma", oh["sigma"][0], "iters", oh["iters"], "status", oh["status"])
tr = hf.trajectory(base[:1], F.NewtonOptions(1e-10, 30, 0))
print("HF trajectory point 0", tr["sigma"][0], tr["iterations"])
print("half bandwidth", hf.half_bandwidth, "n_free", hf.n_free)

import sys, numpy as np
sys.path.insert(0, '.')
import paper_2301_01753_b200 as S
v = int(sys.argv[1]); dims = tuple(int(x) for x in sys.argv[2:5])
y = S.YeeScheme(*dims, 1.0, 0.8, 1.25, 0.2, bc=1)
y.set_variant(v)
rng = np.random.default_rng(0)
y.load(rng.standard_normal(y.n_faces), rng.standard_normal(y.n_edges))
y.advance(int(sys.argv[5]))
print("variant", v, dims, "ok", y.energy())

import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2507_15121_b200 as sk
from paper_2507_15121_b200.distributed import DistributedCpAls
t = sk.synth_tensor_device((300, 200, 100), 400_000, seed=6, unique=False)
fs = sk.random_factors(t.shape, 16, seed=1)
dev_f = [torch.from_numpy(f.data.astype(np.float32)).cuda() for f in fs]
plans = sk.build_all_plans(t, sk.PartitionConfig(devices=2))
als = DistributedCpAls(plans, sk.PlatformConfig(rank=16), rank=0, world=1)
facs, lam, hist = als.run(dev_f, iterations=2)
idx = t.indices.astype(np.int64); vals = t.values.astype(np.float64)
F = [f.double().cpu().numpy() for f in facs]
model = np.ones((len(vals), 16))
for w in range(3): model *= F[w][idx[:, w]]
inner = float(vals @ (model @ lam))
G = np.ones((16, 16))
for f in F: G *= f.T @ f
msq = float(lam @ G @ lam); xsq = float(vals @ vals)
print('hist', hist, 'host fit', 1 - np.sqrt(max(xsq - 2 * inner + msq, 0)) / np.sqrt(xsq), 'xsq', xsq, 'inner', inner, 'msq', msq, 'als xsq', als._x_sq())
model2, _ = sk.cp_als(t, 16, 2, seed=1)
print('cp_als hist', model2.fit_history)

import time, numpy as np, sys
sys.path.insert(0, '.')
import paper_2207_01016_b200 as P
rng = np.random.default_rng(0)
Y = rng.standard_normal((4096, 54)); betas = rng.standard_normal((45, 4096)) * 1e-2
X = rng.standard_normal((2000, 54))
with P.Context(1) as ctx:
    ctx.set_model_dense(Y, betas, 1/54)
    for i in range(50): ctx.model_decision_values_dense(X[i:i+1])
    t0 = time.perf_counter()
    for i in range(1000): ctx.model_decision_values_dense(X[i:i+1])
    t1 = time.perf_counter()
    ctx.model_decision_values_dense(X)
    t2 = time.perf_counter(); ctx.model_decision_values_dense(X); t3 = time.perf_counter()
print(f"K8 per point (one call each): {(t1-t0)/1000*1e6:.1f} us; batched 2000 points: {(t3-t2)*1e3:.2f} ms")

"""Quick GPU sanity run (developer tool): small parity sweep vs the oracle."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle, synth
import paper_1606_05836_b200 as pb

dev = torch.device("cuda:0")
def T(a): return torch.from_numpy(np.ascontiguousarray(a)).to(dev)
worst = 0.0
for n in list(range(1, 21)) + [24]:
    A = synth.gaussian(n, 1000 + n)
    og = oracle.glynn(A).value
    orr = oracle.ryser(A).value
    g = complex(pb.glynn(T(A)).item()); r = complex(pb.ryser(T(A)).item())
    eg = abs(g - og) / abs(og); er = abs(r - orr) / abs(orr)
    worst = max(worst, eg)
    print(f"n={n:2d} glynn rel {eg:.2e}  ryser rel {er:.2e}  plan={pb.plan(n)}", flush=True)
for n in (12, 13):
    for A, name in ((synth.ones(n), "J"), (synth.ones_minus_eye(n), "J-I")):
        ex = oracle.exact(A).value
        g = complex(pb.glynn(T(A)).item()); r = complex(pb.ryser(T(A)).item())
        print(name, n, g == complex(ex[0], ex[1]), r == complex(ex[0], ex[1]), g, float(ex[0]))
As = synth.haar_batch(64, 256, 16, 16, 17)
out = pb.glynn_batched(T(As)).cpu().numpy()
errs = [abs(out[b] - oracle.glynn(As[b]).value) / abs(oracle.glynn(As[b]).value) for b in range(8)]
print("batched max rel", max(errs))
A = synth.gaussian(40, 40)
t0 = time.time(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
pb.glynn(T(synth.gaussian(32, 1)))
torch.cuda.synchronize()
for n in (28, 32, 36):
    A = T(synth.gaussian(n, 1))
    pb.glynn(A); torch.cuda.synchronize()
    e0.record(); v = pb.glynn(A); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    terms = 2 ** (n - 1)
    print(f"n={n} glynn {ms:.3f} ms  {terms / ms * 1e3:.3e} terms/s  alg TFLOP/s {terms * (8 * n - 4) / ms / 1e9:.2f}", flush=True)
print("worst glynn rel", worst)

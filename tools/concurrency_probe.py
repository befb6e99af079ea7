"""How much do two independent DOPRI5 try sequences gain from running concurrently on one GPU
(two contexts / streams / host threads) -- an upper bound on what overlapping the compute-bound
K8 pairs with the memory-bound K3 stages could give.  python tools/concurrency_probe.py [n] [tries]"""
import sys
import threading
import time

import torch

import paper_2309_05331_b200 as rk
import rk_inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
tries = int(sys.argv[2]) if len(sys.argv) > 2 else 20
u0 = torch.from_numpy(rk_inputs.gray_scott_ic(n, n, n, seed=42)).cuda()
sts, ctxs = [], []
for _ in range(2):
    c = rk.Context(0, 1, 0, torch.cuda.Stream())
    s = c.grid(n, n, n, 2)
    s.set_rhs_gray_scott(h=0.0390625)
    s.set(u0)
    torch.cuda.synchronize()
    ctxs.append(c)
    sts.append(s)


def run(s, k):
    for _ in range(k):
        s.try_step("dopri5", 0.0, 0.5, 1e-6, 1e-6)  # dt 0.5: accepted; u advances


for s in sts:
    run(s, 2)
torch.cuda.synchronize()
t0 = time.perf_counter()
run(sts[0], tries)
torch.cuda.synchronize()
t1 = time.perf_counter()
ths = [threading.Thread(target=run, args=(s, tries)) for s in sts]
for t in ths:
    t.start()
for t in ths:
    t.join()
torch.cuda.synchronize()
t2 = time.perf_counter()
one = (t1 - t0) / tries * 1e3
two = (t2 - t1) / (2 * tries) * 1e3
print(f"one stream: {one:.3f} ms/try; two concurrent: {two:.3f} ms/try per try ({one / two:.3f}x)")

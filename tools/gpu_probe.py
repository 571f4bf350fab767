"""GPU probe: FP64 peaks (cuBLAS DGEMM via torch, DMMA/DFMA issue rate) + quick C2 factor timing."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2503_08343_b200 as g
out = {}
dev = torch.device('cuda')
for nn in (4096, 8192):
    a = torch.randn(nn, nn, dtype=torch.float64, device=dev); b = torch.randn(nn, nn, dtype=torch.float64, device=dev)
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    out[f'dgemm_{nn}_tflops'] = 2 * nn**3 / (best * 1e-3) / 1e12
dm, df = g.bench_fp64()
out['dmma_issue_tflops'] = dm; out['dfma_issue_tflops'] = df
print(json.dumps(out))

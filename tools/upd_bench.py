"""Single-tile update latency: tc_gemm_tile (C -= B A^T) via k_update, CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02483_b200._lib import lib, check
for nt in (120, 128, 240):
    a = torch.randn(nt, nt, dtype=torch.float64, device="cuda")
    b = torch.randn(nt, nt, dtype=torch.float64, device="cuda")
    c = torch.randn(nt, nt, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        check("gemm", lib.tc_gemm_tile(a.data_ptr(), b.data_ptr(), c.data_ptr(), nt, s))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    N = 200
    e0.record()
    for _ in range(N):
        check("gemm", lib.tc_gemm_tile(a.data_ptr(), b.data_ptr(), c.data_ptr(), nt, s))
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / N * 1e3
    print(f"nt={nt} tc_gemm_tile {us:.2f} us/launch  ({2*nt**3/us/1e6:.1f} GF/s)")

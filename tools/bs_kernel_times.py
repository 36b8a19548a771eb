"""Dev aid: block-sparse kernel time (ktimer) for one C4 contraction and a 64-batch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench
import paper_2401_01921_b200 as tnb

flush = bench.L2Flush()
c4 = bench.gpu_c4(tnb, 20, 3, flush, bench.Dist())
cb = bench.gpu_c4_batch(tnb, 64, 5, 3, flush, bench.Dist())
print(f"single {c4['bs_gemm_kernel_ms'] * 1e3:.2f} us   batch64 {cb['bs_gemm_kernel_ms']:.4f} ms")

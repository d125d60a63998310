"""Does compute-sanitizer initcheck see TMA (bulk tensor) stores as
initialising?  1: tcgen05 GEMM (C written by TMA tile stores, no split) then a
row-sum kernel reading C; 2: the same with a forced plain-store epilogue."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1605_02688_b200 as T  # noqa: E402

rng = np.random.default_rng(0)
A = rng.standard_normal((512, 512)).astype(np.float32)
B = rng.standard_normal((512, 512)).astype(np.float32)
va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
print("case", os.environ.get("TX_GEMM_NO_TMA_STORE", "tma-store"), flush=True)
T.compile([va, vb], [T.sum(T.dot(va, vb), axis=1)], cuda_graph=False)(A, B)
print("done", flush=True)

"""Small-shape tour of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Never a bench.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1605_02688_b200 as T  # noqa: E402
from oracle import configs as C  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    f32 = "float32"
    # fused elementwise (vector path + ragged tail), broadcast, integer division flag
    g = C.build_ew(T)
    f = T.compile(g["inputs"], g["outputs"], cuda_graph=False)
    f(*C.inputs_ew(100003, seed=1))
    a, b = T.matrix("a", dtype=f32), T.vector("b", dtype=f32)
    T.compile([a, b], [T.tanh(a + b) * 2.0], cuda_graph=False)(rng.standard_normal((37, 29)).astype(np.float32),
                                                               rng.standard_normal(29).astype(np.float32))
    # reductions: rows, columns (TMA-staged), all; max / argmax
    X = rng.standard_normal((1031, 517)).astype(np.float32)
    v = T.matrix("X", dtype=f32)
    for ax in ((0,), (1,), None):
        T.compile([v], [T.sum(v, axis=ax), T.max(v, axis=ax), T.argmax(v, axis=ax)], cuda_graph=False)(X)
    # GEMMs: tcgen05 TF32 (pair / single CTA, split-K), 3xTF32 (promoted), SIMT, skinny
    for (M, N, K) in ((512, 768, 256), (128, 256, 4096), (300, 520, 784), (20, 3000, 600)):
        A = rng.standard_normal((M, K)).astype(np.float32)
        B = rng.standard_normal((K, N)).astype(np.float32)
        va, vb = T.matrix("a", dtype=f32), T.matrix("b", dtype=f32)
        for mode in ("auto", "3xtf32", "simt"):
            T.compile([va, vb], T.dot(va, vb), gemm_mode=mode, cuda_graph=False)(A, B)
    # r02b A-panel multicast (single-CTA tiles, MN-major A, 4-CTA clusters along N)
    At = rng.standard_normal((256, 200)).astype(np.float32)
    Bm = rng.standard_normal((256, 1024)).astype(np.float32)
    va, vb = T.matrix("a", dtype=f32), T.matrix("b", dtype=f32)
    T.compile([va, vb], T.dot(T.transpose(va), vb), cuda_graph=False)(At, Bm)
    # r02 small-M kernel: every B layout, the cluster split of K (DSMEM reduction), an epilogue
    for (M, N, K, tb) in ((20, 200, 800, False), (7, 96, 1000, True), (20, 800, 200, False)):
        A = rng.standard_normal((M, K)).astype(np.float32)
        B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
        bias = rng.standard_normal(N).astype(np.float32)
        va, vb, vc = T.matrix("a", dtype=f32), T.matrix("b", dtype=f32), T.vector("c", dtype=f32)
        T.compile([va, vb, vc], T.tanh(T.dot(va, T.transpose(vb) if tb else vb) + vc), cuda_graph=False)(A, B, bias)
    # r02 rank-3 row-major elementwise form (reversed view, [T] broadcast)
    v3, vt = T.tensor3("X3", dtype=f32), T.vector("t", dtype=f32)
    T.compile([v3, vt], (v3[::-1] + T.dimshuffle(vt, (0, "x", "x"))) * 2.0, cuda_graph=False)(
        rng.standard_normal((5, 6, 36)).astype(np.float32), rng.standard_normal(5).astype(np.float32))
    # training steps: logistic regression (row fusion, skinny GEMMs) and a small MLP
    # (fused epilogues, narrow-grad, stream-K), TF32 and 3xTF32
    gl = C.build_logreg(T)
    x, y = C.inputs_logreg()
    T.compile(gl["inputs"], gl["outputs"], updates=gl["updates"], cuda_graph=False)(x, y)
    for mode in ("auto", "3xtf32"):
        gm = C.build_mlp(T, B=512, H=768)
        xm, ym = C.inputs_mlp(B=512)
        step = T.compile(gm["inputs"], gm["outputs"], updates=gm["updates"], gemm_mode=mode, cuda_graph=False)
        step(xm, ym)
        step(xm, ym)
    # data-parallel step on one rank (bucketed NCCL allreduce on the comm stream)
    from paper_1605_02688_b200.dp import DataParallel
    gd = C.build_mlp(T, B=256, H=256)
    xd, yd = C.inputs_mlp(B=256)
    T.compile(gd["inputs"], gd["outputs"], updates=gd["updates"], cuda_graph=False,
              data_parallel=DataParallel(world_size=1, rank=0, bucket_bytes=1 << 18))(xd, yd)
    # a recurrent step through scan
    h0 = T.vector("h0", dtype=f32)
    W = T.shared((rng.standard_normal((64, 64)) * 0.1).astype(np.float32), name="W")
    xs = T.matrix("xs", dtype=f32)
    hist, _ = T.scan(lambda xt, h: T.tanh(T.dot(h, W) + xt), sequences=[xs], initial_states=[h0])
    T.compile([xs, h0], [T.sum(hist[0] if isinstance(hist, (list, tuple)) else hist)], cuda_graph=False)(
        rng.standard_normal((9, 64)).astype(np.float32), np.zeros(64, np.float32))
    # convolution
    vx, vf = T.tensor4("x", dtype=f32), T.tensor4("f", dtype=f32)
    # r02b implicit-GEMM convolution (stride 1, 32-channel blocks): forward and both gradients
    xi = rng.standard_normal((2, 32, 9, 11)).astype(np.float32)
    fi = rng.standard_normal((8, 32, 3, 3)).astype(np.float32)
    yi = T.conv2d(vx, vf, stride=(1, 1), pad=(1, 1))
    gfi, gxi = T.grad(T.sum(yi * yi), [vf, vx])
    T.compile([vx, vf], [yi, gfi, gxi], cuda_graph=False, conv_impl="gemm")(xi, fi)
    T.compile([vx, vf], [T.conv2d(vx, vf, stride=(2, 2), pad=(1, 1))], cuda_graph=False)(
        rng.standard_normal((2, 3, 11, 9)).astype(np.float32), rng.standard_normal((4, 3, 3, 3)).astype(np.float32))
    print("sanitize tour done")


if __name__ == "__main__":
    main()

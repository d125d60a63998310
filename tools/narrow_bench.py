"""tx_narrow_grad microbenchmark at the MLP's output-layer shape (CUDA events
on one stream; never a bench number): fused vs the three unfused ops.

    python tools/narrow_bench.py [--B 8192] [--H 4096] [--k 10]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=8192)
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_1605_02688_b200 import native
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    B, H, k = a.B, a.H, a.k
    g = torch.Generator(device="cuda").manual_seed(0)
    dz = torch.randn(B, k, device="cuda", generator=g) * 1e-3
    W = torch.randn(H, k, device="cuda", generator=g) * 0.05
    h = torch.tanh(torch.randn(B, H, device="cuda", generator=g))
    dh = torch.empty(B, H, device="cuda")
    gw = torch.empty(H, k, device="cuda")
    db = torch.empty(H, device="cuda")

    def T(t, shape=None, strides=None):
        return native.make_tensor(t.data_ptr(), "float32", t.shape if shape is None else shape,
                                  t.stride() if strides is None else strides)
    tdz, twt, th, tdh, tgw, tdb = T(dz), T(W, (k, H), (1, k)), T(h), T(dh), T(gw), T(db)
    epi = native.TxEpilogue()
    for unfused in (False, True):
        if unfused:
            os.environ["TX_NARROW_UNFUSED"] = "1"
        else:
            os.environ.pop("TX_NARROW_UNFUSED", None)
        wsb = lib.narrow_grad_workspace(tdz, twt, th, tdh, tgw, tdb)
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream

        def run():
            lib.check(lib.lib.tx_narrow_grad(tdz, twt, th, tdh, tgw, ctypes.byref(epi), tdb, 0,
                                             ctypes.c_void_p(ws.data_ptr()), wsb, ctypes.c_void_p(st)))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(a.reps):
            run()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / a.reps * 1e3
        ref_dh = (dz @ W.T) * (1 - h * h)
        ref_gw = h.double().T @ dz.double()
        err_dh = ((dh - ref_dh).abs().max() / ref_dh.abs().max()).item()
        err_gw = ((gw.double() - ref_gw).abs().max() / ref_gw.abs().max()).item()
        err_db = ((db.double() - ref_dh.double().sum(0)).abs().max() / ref_dh.abs().sum(0).max()).item()
        gbs = 2 * B * H * 4 / (us * 1e-6) / 1e9
        print(f"{'unfused' if unfused else 'fused  '} B={B} H={H} k={k}: {us:7.1f} us  "
              f"({gbs:.0f} GB/s of the 2*B*H*4 algorithmic bytes)  err dh {err_dh:.1e} gW {err_gw:.1e} db {err_db:.1e}")


if __name__ == "__main__":
    main()

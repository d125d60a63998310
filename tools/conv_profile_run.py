"""One 3x3 conv layer training step (bench conv shape) for ncu launch lists (never a bench number)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1605_02688_b200 as T
from tools.ref_bench import conv_graph, conv_inputs
x, f0 = conv_inputs()
ins, outs, ups = conv_graph(T, f0)
fn = T.compile(ins, outs, updates=ups, conv_impl="gemm")
xd = torch.from_numpy(x).cuda()
for _ in range(2):
    fn.call_device(xd, sync=True)

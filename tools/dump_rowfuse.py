"""Print the generated row-fusion kernels of the logreg / MLP steps (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_02688_b200 as T  # noqa: E402
from oracle import configs as C  # noqa: E402

torch.cuda.set_device(0)
g = C.build_logreg(T)
f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
x, y = C.inputs_logreg()
f(x, y)
plan = next(iter(f._plans.values()))
for src in plan.row_sources:
    print(src)

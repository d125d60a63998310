"""Host-side cost of one logistic-regression call through the public API
(diagnostic): cProfile over 300 calls, plus wall time per call."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_02688_b200 as T  # noqa: E402
from oracle import configs as C  # noqa: E402

g = C.build_logreg(T)
f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
x, y = C.inputs_logreg()
for _ in range(20):
    f(x, y)
t0 = time.perf_counter()
for _ in range(300):
    f(x, y)
print("us per call", (time.perf_counter() - t0) / 300 * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    f(x, y)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

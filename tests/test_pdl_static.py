"""Programmatic dependent launch is only safe when every kernel launched with
the attribute waits for its predecessor before touching memory
(tx_common.h TX_GRID_WAIT).  Static check over the CUDA sources (no GPU):
every __global__ kernel opens with TX_GRID_WAIT() -- or, in the NVRTC
templates and the generated row kernels, with griddepcontrol.wait -- and no
kernel is launched with the <<<>>> syntax (which would bypass tx::launch)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1605_02688_b200", "csrc")


def _kernel_bodies(src):
    for m in re.finditer(r"__global__", src):
        depth, k = 0, m.start()
        while True:
            ch = src[k]
            if ch == "(":
                depth += 1
            elif ch == ")":
                depth -= 1
            elif ch == ";" and depth == 0:
                k = -1
                break
            elif ch == "{" and depth == 0:
                break
            k += 1
        if k < 0:
            continue
        names = [n for n in re.findall(r"(\w+)\s*\(", src[m.start():k]) if n != "__launch_bounds__"]
        name = names[0] if names else "?"
        yield name, src[k + 1:k + 400]


def test_every_kernel_waits_first():
    checked = 0
    for fn in sorted(os.listdir(CSRC)):
        if not fn.endswith((".cu", ".cuh")):
            continue
        src = open(os.path.join(CSRC, fn)).read()
        for name, body in _kernel_bodies(src):
            first = body.strip().splitlines()[0].strip()
            assert first.startswith("TX_GRID_WAIT()") or "griddepcontrol.wait" in first, (fn, name, first)
            checked += 1
    assert checked >= 35  # every kernel of the library (38 in r02)


def test_no_triple_chevron_launches():
    for fn in sorted(os.listdir(CSRC)):
        if fn.endswith((".cu", ".cuh")):
            assert "<<<" not in open(os.path.join(CSRC, fn)).read(), fn


def test_generated_row_kernels_wait_first():
    from paper_1605_02688_b200 import rowfuse
    assert "griddepcontrol.wait" in rowfuse._GRID_WAIT
    src = open(os.path.join(ROOT, "paper_1605_02688_b200", "rowfuse.py")).read()
    assert src.count("_GRID_WAIT,") >= 2

"""The megakernel must stay (nearly) spill-free: a 10-warp CTA is capped at 168
registers, and 216 bytes of local-memory spills around the GEMV loop cost ~12%
of decode time (measured this round).  A few bytes in once-per-task code
(routing, slot decoding) are tolerated.  Reads the ptxas report of the in-tree
build (Makefile: build/cu/megakernel.ptxas.txt)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPORT = os.path.join(ROOT, "build", "cu", "megakernel.ptxas.txt")


@pytest.mark.skipif(not os.path.exists(REPORT), reason="megakernel not built in-tree")
def test_persistent_kernels_do_not_spill():
    text = open(REPORT).read()
    found = {}
    for m in re.finditer(r"Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, "
                         r"(\d+) bytes spill loads", text):
        found[m.group(1)] = (int(m.group(3)), int(m.group(4)))
    kernels = {k: v for k, v in found.items() if "et_static_kernel" in k or "et_dynamic_kernel" in k}
    # <kMoE, kTC> instantiations of each scheduler: dense, MoE, tensor-core, MoE + tensor-core
    assert len(kernels) == 8, found
    for name, (st, ld) in kernels.items():
        if "ILb0ELb0E" in name and "static" in name:  # dense mma.sync instantiation (the Llama bs=1 decode path)
            assert st == 0 and ld == 0, (name, st, ld)
        elif "ILb0ELb0E" in name:  # its dynamic-scheduler twin: a few bytes around the completion path
            assert st <= 32 and ld <= 32, (name, st, ld)
        else:  # bounded (once-per-task routing / slot decoding / epilogue code)
            assert st <= 384 and ld <= 384, (name, st, ld)
    # the tensor-core streaming loops (issuer, producer) are register-resident everywhere
    for name, (st, ld) in found.items():
        if "tc_issue" in name or "tc_produce" in name:
            assert st == 0 and ld == 0, (name, st, ld)

"""Build-free driver of tests/cpp/dropin_trace.cpp (compiled to scratch_libs/dropin_trace): the C2 batch file, then the timeline."""
import sys, os, subprocess; sys.path.insert(0,'.')
import numpy as np
from paper_2106_14995_b200 import synth
b = synth.branch(65536, 6)
path = "/tmp/c2.bin"
with open(path, "wb") as fh:
    fh.write(np.array([b.count, 6, b.params.shape[1]], dtype=np.int64).tobytes())
    for arr in (b.x0, b.lower, b.upper, b.params): fh.write(np.ascontiguousarray(arr, dtype=np.float64).tobytes())
print(subprocess.run(["scratch_libs/dropin_trace", path], capture_output=True, text=True).stdout)

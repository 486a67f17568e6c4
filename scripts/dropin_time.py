"""End-to-end time of C++ drop-in builds on the C2 batch (interleaved):
python scripts/dropin_time.py exe1 [exe2 ...]"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2106_14995_b200 import synth  # noqa: E402

b = synth.branch(65536, 6)
path = f"/tmp/tb_c2_batch_{os.getpid()}.bin"
with open(path, "wb") as fh:
    fh.write(np.array([b.count, 6, b.params.shape[1]], dtype=np.int64).tobytes())
    for arr in (b.x0, b.lower, b.upper, b.params):
        fh.write(np.ascontiguousarray(arr, dtype=np.float64).tobytes())
for r in range(3):
    for exe in sys.argv[1:]:
        out = subprocess.run([exe, path, "9"], capture_output=True, text=True, timeout=300)
        print(f"{os.path.basename(exe):26s} {out.stdout.strip() or out.stderr[-400:]}", flush=True)
os.remove(path)

"""Driver for targeted ncu captures: one warm step of a BASELINE config, then
the region of interest between cudaProfilerStart/Stop, so that
`ncu --profile-from-start off -k regex:<kernel> -c <n>` captures exactly it.

    python tools/prof_driver.py --config 3 --what apply|step
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5863_b200 as pb  # noqa: E402

MODES = {1: ("c+e+f", 10.0, 15, False), 2: ("adaptive", 10.0, 10, False), 3: ("adaptive", 5.0, 15, False),
         4: ("adaptive", 10.0, 15, True), 5: ("adaptive", 10.0, 15, False)}

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--what", default="apply", choices=["apply", "step"])
a = ap.parse_args()
cudart = ctypes.CDLL("libcudart.so") if False else None
try:
    import torch  # noqa: F401  (cudaProfilerStart through torch's runtime)
    start, stop = torch.cuda.profiler.start, torch.cuda.profiler.stop
except Exception:  # pragma: no cover
    start = stop = lambda: None
b = pb.BDDC(config=a.config)
mode, tau, maxv, bf = MODES[a.config]
b.step(mode, tau, maxv, base_faces=bf)
b.operator_times(2)
start()
if a.what == "apply":
    b.operator_times(1)
else:
    b.step(mode, tau, maxv, base_faces=bf)
stop()
print("done", a.config, a.what)

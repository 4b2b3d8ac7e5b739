"""Times run_phase_experiment (the reference CLI's panels, msfft_main.cpp:
212-216, SNR list -20,-10,0,20, 200 trials) on the GPU and with the
reference's own CPU code; windows are designed in an untimed warm-up call on
both sides.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200.signal as S  # noqa: E402
from oracle import load  # noqa: E402

R = load("reference")
panels = {"a": (8192, 50, 32), "b": (131072, 50, 2048), "c": (1048576, 50, 2048),
          "d": (4194304, 50, 8192)}
snrs, trials = [-20.0, -10.0, 0.0, 20.0], int(os.environ.get("TRIALS", "200"))
res = {"snr_list": snrs, "trials": trials}
for name in os.environ.get("PANELS", "abcd"):
    n, k, L = panels[name]
    b = n // L
    S.run_phase_experiment(n, k, b, snrs, 1, 1)
    R.phase_experiment(n, k, b, snrs, 1, 1)
    t0 = time.perf_counter()
    g = S.run_phase_experiment(n, k, b, snrs, trials, 1)
    g_ms = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    r = R.phase_experiment(n, k, b, snrs, trials, 1)
    c_ms = (time.perf_counter() - t0) * 1e3
    res[name] = {"n": n, "k": k, "L": L, "gpu_ms": g_ms, "cpu_ms": c_ms,
                 "bins_identical": all(np.array_equal(x.bin_mass, y["bin_mass"]) for x, y in zip(g, r)),
                 "max_p50_rel_diff": max(abs(x.p50 - y["p50"]) / y["p50"] for x, y in zip(g, r))}
    print(json.dumps({name: res[name]}), flush=True)
print(json.dumps(res))

"""AMG hierarchy setup time, device vs host, for PMIS with direct and MM-ext
interpolation (not a test): python tools/probe_mmext_setup.py [SPEC]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
ilug.Hierarchy(ilug.Matrix.generate("poisson3d(32,32,32)"),  # warm-up: CUDA context, module load
               ilug.Config().update({"amg.coarsening": "pmis", "device.amg_setup": "device"}), host_only=True)
A = ilug.Matrix.generate(spec)
for interp in ("direct", "mm_ext"):
    for where in ("device", "host"):
        kv = {"amg.coarsening": "pmis", "amg.interpolation": interp, "device.amg_setup": where}
        t = time.time()
        H = ilug.Hierarchy(A, ilug.Config().update(kv), host_only=True)
        print(f"{spec} {interp:7s} {where:6s} levels {H.levels:2d}  {time.time() - t:6.2f} s", flush=True)
        del H

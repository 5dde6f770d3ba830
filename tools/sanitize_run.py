"""Small run of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2605_13766_b200 as er
for name, n in (("cfg2", 24), ("cfg5", 6), ("cfg4", 8)):
    w = W.make(name, n_rods=n)
    for kernel in (0, 1, 2):
        with er.RodBatch(w) as b:
            b.set_option(er.ER_OPT_KERNEL, kernel)
            b.step(3, w.dt)
            b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, 4)
            b.step(8, w.dt)
            b.diagnostics()
            b.get_state()
print("sanitize run ok")

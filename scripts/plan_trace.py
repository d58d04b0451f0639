"""Planner phase times (EARL_PLAN_TRACE=1 prints them from the library) for the configs' N."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_05943_b200 import workloads as W  # noqa: E402
from paper_2510_05943_b200.dispatch import EmulatedDispatch  # noqa: E402

ed = EmulatedDispatch(8)
for name, lens, cfg in [("c3", W.c2_lengths(0), "c3"), ("c2-lpt", W.c2_lengths(0), "c2-lpt"),
                        ("c4", W.c4_lengths(0), "c4"), ("c0", np.zeros(512, np.int64), "c3")]:
    src, dst = W.config_layouts(cfg, 8, len(lens))
    d = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
    p = ed.plan(src, dst, d, W.field_set("scalar6-fp32"))
    for _ in range(3):
        print(name, file=sys.stderr, end=" ")
        p.replan(d)
    torch.cuda.synchronize()
    p.destroy()

"""In-situ per-op time breakdown of one full C2 forward (eager replay, CUDA
events around every C-ABI call), grouped by op and by member count.

    python scripts/step_breakdown.py [--segments 128] [--schedule diagonal]
"""

import argparse
import collections
import json
import os
import sys

# per-op events are recorded on the current stream: time the one-stream issue order
os.environ.setdefault("ARMT_DUAL", "0")

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2506_05229_b200 import ModelConfig  # noqa: E402
from paper_2506_05229_b200.engine import prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import Session  # noqa: E402

GEMM_NAMES = {0: "store", 1: "residual", 2: "retrieve", 3: "swiglu", 4: "rope", 5: "lse", 6: "qproj_dpfp"}


class Proxy:
    def __init__(self, lib, log):
        self.lib, self.log = lib, log

    def __getattr__(self, name):
        fn = getattr(self.lib, name)
        if not name.startswith("armt_") or name in ("armt_last_error", "armt_fold_workspace_bytes",
                                                    "armt_fold_tc_workspace_bytes", "armt_memop_rows"):
            return fn

        def wrapped(*a):
            key = name
            if name == "armt_gemm":
                args = a[0]
                key = f"gemm_{GEMM_NAMES.get(args.epilogue, args.epilogue)}_N{args.N}_K{args.K}"
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = fn(*a)
            e1.record()
            G = getattr(a[0], "G", None) if a and hasattr(a[0], "G") else None
            self.log.append((key, G, e0, e1))
            return rc
        return wrapped


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--segments", type=int, default=128)
    ap.add_argument("--schedule", default="diagonal")
    args = ap.parse_args()
    cfg = ModelConfig(**bench.C2, eps_assoc=bench.EPS_ASSOC, seed=0)
    n = args.segments * cfg.segment_size
    w = bench.make_weights(cfg, "device")
    prep = prepare_weights(w, "bf16")
    del w
    sess = Session(prep, n, schedule=args.schedule, graph=False)
    tokens = torch.as_tensor(np.random.default_rng([0, n]).integers(0, cfg.vocab_size, n)).cuda()
    sess.forward(tokens)
    torch.cuda.synchronize()
    log = []
    eng = sess.runner.engine
    eng.lib = Proxy(eng.lib, log)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sess.forward(tokens)
    b.record()
    torch.cuda.synchronize()
    total = a.elapsed_time(b)
    by_op = collections.defaultdict(float)
    by_op_full = collections.defaultdict(float)
    for key, G, e0, e1 in log:
        t = e0.elapsed_time(e1)
        by_op[key] += t
        if G == sess.plan.max_members:
            by_op_full[key] += t
    acc = sum(by_op.values())
    print(json.dumps({"total_ms": total, "sum_ops_ms": acc, "launch_gaps_ms": total - acc}))
    for k, v in sorted(by_op.items(), key=lambda x: -x[1]):
        print(f"{v:9.2f} ms {100 * v / total:5.1f}%  (full-width steps {by_op_full.get(k, 0):8.2f} ms)  {k}")


if __name__ == "__main__":
    main()

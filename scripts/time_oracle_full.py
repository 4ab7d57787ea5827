"""Time the FP64 oracle (oracle/, plain C + OpenMP across independent layers/factors) on a FULL
workload once -- every layer of the config, one cold K-FAC update: factors, eigendecomposition of
every factor, preconditioning (Eqs. 13-15), KL-clip -- and write the per-stage wall times to
profiles/oracle_full_<config>.json.  bench.py's cpu_baseline / --impl reference extrapolate a bounded
layer sample to the full workload; this file is the measured cross-check of that extrapolation.

Calls only oracle/ and workloads/ (seeded inputs); no CUDA.
Usage: python scripts/time_oracle_full.py [r50]
"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import shapes  # noqa: E402
from workloads.gen import layer_inputs  # noqa: E402


def main(cfg):
    layers = shapes.layers_for(cfg)
    hp = shapes.HPARAMS[cfg]
    oracle.build()
    t_gen = time.perf_counter()
    acts, gouts, grads = layer_inputs(layers, seed=0)
    t0 = time.perf_counter()
    A, G = oracle.update_factors(layers, acts, gouts, xi=hp["xi"], first=True)
    t1 = time.perf_counter()
    Qs, vs = oracle.symeig_batch(A + G)
    t2 = time.perf_counter()
    n = len(layers)
    P = oracle.precondition_batch(grads, Qs[n:], vs[n:], Qs[:n], vs[:n], hp["damping"])
    _, nu, s = oracle.kl_clip(P, grads, hp["lr"], hp["kappa"])
    t3 = time.perf_counter()
    cpu = "?"
    try:
        cpu = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        pass
    out = {"config": cfg, "layers": n, "batch_per_gpu": layers[0].batch,
           "stages_s": {"factors": t1 - t0, "eigen": t2 - t1, "precond_klclip": t3 - t2},
           "total_s": t3 - t0, "input_generation_s": t0 - t_gen, "nu": nu, "s": s,
           "cores": len(os.sched_getaffinity(0)), "cpu": cpu, "host": platform.node(),
           "how": "oracle.full-step stages on every layer (OpenMP across layers/factors), wall clock"}
    path = os.path.join(ROOT, "profiles", f"oracle_full_{cfg}.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r50")

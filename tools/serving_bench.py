"""Serving end to end through the UNMODIFIED reference InferenceService
(serving/service.py, "baseline" security preset = empty chain), GPU model vs the
reference CPU model: client-side p50/p99 request latency (submit -> resolved
future, nearest rank, telemetry/metrics.py:33-37) and rows/s, at several
request sizes.  Needs baseline/_ref (tools/install_reference.sh).
    python tools/serving_bench.py [precision] > profiles/serving_r2.json
"""
import json
import sys
import time
import uuid
from concurrent.futures import wait
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
import paper_2510_19689_b200 as P  # noqa: E402
from paper_2510_19689_b200 import workloads as W  # noqa: E402
from tabserve.model.config import ModelConfig  # noqa: E402
from tabserve.model.network import TabNetModel as RefModel  # noqa: E402
from tabserve.security.chain import SecurityChain, SecurityChainConfig  # noqa: E402
from tabserve.serving.batching import BatcherConfig, InferenceRequest  # noqa: E402
from tabserve.serving.service import InferenceService  # noqa: E402


def nearest_rank(v, q):
    s = sorted(v)
    return s[max(1, int(np.ceil(q / 100 * len(s)))) - 1]


def run(model, rows_per_req, n_req, concurrency, max_batch):
    svc = InferenceService(model, SecurityChain(SecurityChainConfig.preset("baseline")),
                           batcher=BatcherConfig(max_batch=max_batch, max_delay_ms=1.0, queue_capacity=100000),
                           parallelism=2).start()
    x = W.make_inputs(W.WORKLOADS["hr"], rows_per_req * 64).astype(np.float64)
    lat = []
    try:
        # warm-up: sequential, then at the timed concurrency, so the batch sizes the
        # timed phase forms have been seen once (one-time staging growth per host
        # context: page-locking memory costs ~0.1 s on this VM)
        for _ in range(20):
            svc.submit(InferenceRequest(str(uuid.uuid4()), x[:rows_per_req])).future.result(timeout=60)
        for _ in range(3):
            fs = [svc.submit(InferenceRequest(str(uuid.uuid4()), x[i * rows_per_req:(i + 1) * rows_per_req])).future
                  for i in range(min(64, 2 * concurrency))]
            for f in fs:
                f.result(timeout=60)
        t_start = time.perf_counter()
        inflight = []
        sent = 0
        while sent < n_req or inflight:
            while sent < n_req and len(inflight) < concurrency:
                i = sent % 64
                t0 = time.perf_counter()
                tk = svc.submit(InferenceRequest(str(uuid.uuid4()), x[i * rows_per_req:(i + 1) * rows_per_req]))
                tk.future.add_done_callback(lambda f, t0=t0: lat.append(1e3 * (time.perf_counter() - t0)))
                inflight.append(tk.future)
                sent += 1
            done, _ = wait(inflight, return_when="FIRST_COMPLETED")
            inflight = [f for f in inflight if f not in done]
        el = time.perf_counter() - t_start
    finally:
        svc.stop()
    return {"rows_per_request": rows_per_req, "requests": n_req, "concurrency": concurrency,
            "p50_ms": nearest_rank(lat, 50), "p99_ms": nearest_rank(lat, 99),
            "rows_per_s": n_req * rows_per_req / el, "errors": svc.error_responses}


def main():
    prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
    base = W.make_model("hr", "trained")
    gpu = P.TabNetModel.from_reference(base, precision=prec)
    c = base.config
    cpu = RefModel(config=ModelConfig(feature_count=c.feature_count, n_classes=c.n_classes, n_d=c.n_d,
                                      n_a=c.n_a, n_steps=c.n_steps, gamma=c.gamma),
                   params=base.params, norm_mean=base.norm_mean, norm_var=base.norm_var,
                   model_version=base.model_version)
    out = {"service": "tabserve InferenceService (unmodified), preset 'baseline', parallelism 2, max_delay 1 ms",
           "precision": prec, "results": []}
    for rows, conc, n in ((1, 1, 400), (1, 32, 2000), (16, 32, 2000), (256, 8, 400)):
        for arm, model in (("gpu", gpu), ("reference_cpu", cpu)):
            nn = n if arm == "gpu" else max(40, n // 10)
            r = run(model, rows, nn, conc, max_batch=max(256, rows))
            r["arm"] = arm
            out["results"].append(r)
            print(json.dumps(r), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

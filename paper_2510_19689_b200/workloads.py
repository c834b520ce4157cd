"""Synthetic workloads of BASELINE.json's configs.

Shapes ``(F, n_d, n_a, n_steps, n_classes)``; weights from the reference's own
seeded ``init_parameters`` (network.py:71-97, mirrored in ``network.py`` here)
in two regimes, inputs ``x ~ N(0,1)`` drawn in float32 so that the GPU path and
the float64 oracle see bit-identical values.  Nothing here touches the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import ModelConfig


@dataclass(frozen=True)
class Workload:
    name: str
    config_id: int
    feature_count: int
    n_d: int
    n_a: int
    n_steps: int
    n_classes: int
    batch: int
    description: str
    regression: bool = False     # evaluated through TabNetRegressor (identity head on column 0)
    shard: bool = False          # bench default: the batch is row-sharded over the ranks (strong scaling)

    def model_config(self, seed: int = 0) -> ModelConfig:
        return ModelConfig(feature_count=self.feature_count, n_classes=self.n_classes,
                           n_d=self.n_d, n_a=self.n_a, n_steps=self.n_steps, seed=seed)


# BASELINE.json "configs" in order.  BLS is a regression in BASELINE.json; the
# reference has no regression head (config.py:32-33), so the workload's weights
# are the 2-class reference model and the engine runs TabNetRegressor, the
# identity head on its logit column 0.
WORKLOADS: dict[str, Workload] = {
    "adult": Workload("adult", 0, 14, 8, 8, 3, 2, 4096,
                      "Adult-shaped (14 features, n_d=n_a=8, n_steps=3, binary) batch 4,096"),
    "hr": Workload("hr", 1, 35, 16, 16, 5, 2, 65536,
                   "HR-attrition-shaped (35 features, n_d=n_a=16, n_steps=5) batch 65,536, with feature masks"),
    "bls": Workload("bls", 2, 64, 32, 32, 5, 2, 262144,
                    "BLS-shaped synthetic regression (64 features, n_d=n_a=32, n_steps=5) batch "
                    "262,144, row-sharded", regression=True, shard=True),
    "hr_latency": Workload("hr_latency", 3, 35, 16, 16, 5, 2, 1024,
                           "HR shape latency sweep batch 1-1,024"),
    "wide": Workload("wide", 4, 512, 64, 64, 8, 10, 1 << 24,
                     "wide TabNet (512 features, n_d=n_a=64, n_steps=8, 10 classes) 16M rows", shard=True),
    # the north-star target: HR batch 65,536 row-sharded over the GPUs of one box
    "hr8": Workload("hr8", 1, 35, 16, 16, 5, 2, 65536,
                    "HR-attrition-shaped (35 features, n_d=n_a=16, n_steps=5) batch 65,536 row-sharded "
                    "over the ranks (north star: 8xB200)", shard=True),
}

ATT_SCALE_TRAINED = 16.0   # SURVEY.md §8(d) "trained-like": step*_att_W x16
HEAD_SCALE_TRAINED = 8.0   #                                  head_W x8


def make_params(w: Workload, regime: str = "trained", seed: int = 0) -> dict[str, np.ndarray]:
    from .network import init_parameters
    params = init_parameters(w.model_config(seed))
    if regime == "trained":
        for k in list(params):
            if k.endswith("_att_W"):
                params[k] = params[k] * ATT_SCALE_TRAINED
        params["head_W"] = params["head_W"] * HEAD_SCALE_TRAINED
    elif regime != "init":
        raise ValueError(f"unknown weight regime {regime!r}")
    return params


def make_norm_stats(w: Workload, seed: int = 7) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(seed)
    mean = rng.standard_normal(w.feature_count)
    var = rng.uniform(0.5, 2.0, w.feature_count)
    return mean, var


INPUT_BLOCK = 65536   # rows per independently seeded block of the input stream


def make_inputs(w: Workload, rows: int, seed: int | None = None, start: int = 0) -> np.ndarray:
    """float32 N(0,1) rows ``[start, start+rows)`` of the workload's stream.

    The stream is cut into blocks of ``INPUT_BLOCK`` rows, block b drawn from
    its own generator (block 0 from ``default_rng(seed)``, so the first 65,536
    rows are the plain ``default_rng(seed).standard_normal`` draw the golden
    fixtures hold; block b > 0 from ``default_rng([seed, b])``).  A shard at a
    large offset therefore costs only its own rows."""
    base = 1000 + w.config_id if seed is None else seed
    f = w.feature_count
    out = np.empty((rows, f), dtype=np.float32)
    if rows <= 0:
        return out
    for b in range(start // INPUT_BLOCK, (start + rows - 1) // INPUT_BLOCK + 1):
        lo, hi = max(start, b * INPUT_BLOCK), min(start + rows, (b + 1) * INPUT_BLOCK)
        rng = np.random.default_rng(base) if b == 0 else np.random.default_rng([base, b])
        blk = rng.standard_normal((hi - b * INPUT_BLOCK, f), dtype=np.float32)   # prefix of the block
        out[lo - start:hi - start] = blk[lo - b * INPUT_BLOCK:]
    return out


def make_engine_model(name: str, regime: str = "trained", *, precision: str = "auto",
                      device: int | None = None):
    """The engine model a workload runs: TabNetModel, or TabNetRegressor for the
    regression workload (BLS)."""
    from .network import TabNetModel, TabNetRegressor
    cls = TabNetRegressor if WORKLOADS[name].regression else TabNetModel
    return cls.from_reference(make_model(name, regime), precision=precision, device=device)


def make_model(name: str, regime: str = "trained", *, model_cls=None):
    """A TabNetModel (this package's, or ``model_cls``) for a named workload."""
    from .network import TabNetModel
    w = WORKLOADS[name]
    cls = model_cls or TabNetModel
    mean, var = make_norm_stats(w)
    return cls(config=w.model_config(), params=make_params(w, regime),
               norm_mean=mean, norm_var=var, model_version=f"{name}-{regime}-v1")


def algorithmic_counts(w: Workload) -> dict:
    """Per-row algorithmic FLOPs and HBM bytes.
    A regression head (C=1) writes its one output value and no class."""
    f, nd, na, s = w.feature_count, w.n_d, w.n_a, w.n_steps
    h = nd + na
    c = 1 if w.regression else w.n_classes
    out_b = 4 if w.regression else 8 * c + 4              # logits (+ probs + class)
    flops = 2 * ((s + 1) * (2 * h * f + 6 * h * h) + s * na * f + nd * c)
    bytes_pe = 4 * f + 4 * s * f + 4 * f + out_b          # x, masks, importance, head outputs
    bytes_po = 4 * f + out_b                              # predict-only
    return dict(flops_per_row=flops, bytes_per_row=bytes_pe, bytes_per_row_predict=bytes_po)

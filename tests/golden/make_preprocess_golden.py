"""Golden fixtures for device preprocessing from the
UNMODIFIED reference ETL (data/synth.py, data/ingest.py, data/preprocess.py).

Run in the builder container (where /root/reference exists):

    python tests/golden/make_preprocess_golden.py

For HR and Adult: fit a PreprocessPlan on one synthetic table, then transform a
second table (other seed, extra missing cells and unseen category levels) with
the reference's PreprocessPlan.transform (preprocess.py:68-122).  Stores the
plan (to_dict), the raw columns of the second table and the reference's
float64 matrix / column names / unseen counts.  Only the .npz travels.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    from tabserve.data import ingest, preprocess, schema, synth

    out = {}
    for name, gen, sch, rows in (("hr", synth.generate_hr_csv, schema.hr_schema(), 3000),
                                 ("adult", synth.generate_adult_csv, schema.adult_schema(), 3000)):
        fit_tab = ingest.ingest_csv(gen(rows=rows, seed=0), sch)
        plan = preprocess.fit_preprocess(fit_tab, sch)
        tab = ingest.ingest_csv(gen(rows=700, seed=1), sch)
        rng = np.random.default_rng(5)
        # extra missing cells and unseen levels in the feature columns
        for t in plan.transforms:
            col = tab.columns[t.label]
            for i in rng.choice(len(col), 12, replace=False):
                col[i] = None
            if t.kind in ("onehot", "ordinal"):
                for i in rng.choice(len(col), 5, replace=False):
                    col[i] = "never-seen-level"
        res = plan.transform(tab)
        cols = {t.label: tab.columns[t.label] for t in plan.transforms}
        out[f"{name}__plan"] = np.array(json.dumps(plan.to_dict()))
        out[f"{name}__columns"] = np.array(json.dumps(cols))
        out[f"{name}__rows"] = np.array(tab.n_rows)
        out[f"{name}__matrix"] = res.matrix.values
        out[f"{name}__names"] = np.array(json.dumps(res.matrix.column_names))
        out[f"{name}__unseen"] = np.array(json.dumps(res.unseen_counts, sort_keys=True))
        print(name, res.matrix.values.shape, res.unseen_counts)
    np.savez_compressed(OUT / "preprocess.npz", **out)


if __name__ == "__main__":
    main()

"""Golden fixtures (tests/golden/, generated from the reference by make_golden.py).

CPU: the oracle build still reproduces them (pins the oracle), and the product's plan
builder reproduces every schedule bit-exactly. GPU: the product's renders match the
reference's batched and per-node outputs within rel-L-inf 1e-4.
"""
import json
import os

import numpy as np
import pytest

from conftest import cuda_ok

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-4


def load_schedules():
    with open(os.path.join(HERE, "schedules.json")) as f:
        return json.load(f)


def load_renders():
    d = np.load(os.path.join(HERE, "renders.npz"))
    cases = []
    for i in range(int(d["count"][0])):
        params = {int(k[len(f"c{i}_p"):]): d[k] for k in d.files if k.startswith(f"c{i}_p")}
        cases.append(dict(types=d[f"c{i}_types"], edges=d[f"c{i}_edges"], fs=float(d[f"c{i}_meta"][0]),
                          params=params, src=d[f"c{i}_src"], out=d[f"c{i}_out"],
                          slow=d[f"c{i}_slow"] if f"c{i}_slow" in d.files else None))
    return cases


def as_steps(rd):
    return [[int(s.type), s.param_begin, s.param_end, s.store_begin, s.store_end, s.gather, s.aggregate] for s in rd.steps]


def test_product_schedules_match_golden(mg):
    for c in load_schedules():
        fg = mg.to_flat(mg.Graph.from_arrays(c["types"], c["edges"]))
        rd = mg.compute_render_data(fg, c["strategy"])
        assert rd.schedule.type_codes() == c["type_codes"], c["name"]
        assert rd.schedule.subsets == c["subsets"]
        assert rd.sigma == c["sigma"]
        assert as_steps(rd) == c["steps"]
        assert {str(int(k)): v for k, v in rd.param_source_rows.items()} == c["param_source_rows"]


def test_oracle_reproduces_golden(ref):
    for c in load_schedules()[:12]:
        p = ref.Plan(np.array(c["types"]), np.array(c["edges"]), c["strategy"])
        assert p.type_codes == c["type_codes"] and p.subsets == c["subsets"] and p.sigma == c["sigma"]
    for c in load_renders():
        out = ref.Plan(c["types"], c["edges"], 1).render(c["params"], c["src"], sample_rate=c["fs"])
        assert ref.rel_linf(out, c["out"]) < 1e-12


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_product_renders_match_golden(mg):
    from oracle.ref import rel_linf
    for c in load_renders():
        fg = mg.to_flat(mg.Graph.from_arrays(c["types"], c["edges"]))
        rd = mg.compute_render_data(fg)
        procs = mg.ProcessorSet(sample_rate=c["fs"])
        got = mg.render(rd, procs, rd.reorder_params(c["params"]), c["src"])
        assert rel_linf(got, c["out"]) < TOL
        if c["slow"] is not None:
            assert rel_linf(got, c["slow"]) < TOL

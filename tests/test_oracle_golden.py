"""The CPU oracle against the reference's recorded outputs (parity pin)."""

import numpy as np
import pytest

import oracle
from golden_util import TABLE_PARAMS, case_input, digest

SMALL = ["ref_random_multilayer_s9", "ref_flat_plane_s7", "ref_spiral_s3",
         "ref_ramp_over_tunnel_s6", "synth_cfg0", "synth_cfg4", "synth_two_storey_small"]


@pytest.mark.parametrize("name", SMALL)
def test_oracle_matches_reference(golden, name):
    case = golden["cases"][name]
    xyz = case_input(name, case)
    t = oracle.build(xyz, case["d_s"], case["r_g"])
    assert list(t["ground"].shape) == case["shape"]
    assert [float(h) for h in t["heights"]] == case["heights"]
    assert list(t["origin"]) == case["origin"]
    assert digest(t["ground"]) == case["ground_sha256"]
    assert digest(t["ceiling"]) == case["ceiling_sha256"]
    cost = oracle.evaluate(t["ground"], t["ceiling"], case["r_g"], TABLE_PARAMS)
    assert digest(cost) == case["cost_sha256"]
    assert oracle.simplify(t["ground"], cost) == case["keep"]


@pytest.mark.slow
@pytest.mark.parametrize("name", ["synth_cfg1"])
def test_oracle_matches_reference_large(golden, name):
    test_oracle_matches_reference(golden, name)


def test_oracle_inflation_cases(golden):
    for c in golden["inflation"]:
        w = oracle.kernel_weights(0.2, 0.4, c["r_g"])
        assert digest(w) == c["kernel_sha256"]
        shape = tuple(c["shape"])
        g = np.random.default_rng(c["seed"]).uniform(0.0, 50.0, shape).astype(np.float32)
        g[np.random.default_rng(c["seed"] + 1).uniform(size=shape) < 0.03] = 50.0
        assert digest(oracle.inflate(g, w)) == c["out_sha256"]


@pytest.mark.parametrize("name", ["ref_random_multilayer_s9", "ref_spiral_s3", "synth_cfg0"])
def test_oracle_lga_bytes_match_reference(golden, name):
    """The LGA archive restatement reproduces the reference's archive bytes."""
    import hashlib
    from oracle.archive import lga_bytes
    case = golden["cases"][name]
    t = oracle.build(case_input(name, case), case["d_s"], case["r_g"])
    cost = oracle.evaluate(t["ground"], t["ceiling"], case["r_g"], TABLE_PARAMS)
    args = (t["heights"], t["origin"], case["r_g"], t["z_min"], case["d_s"])
    built = lga_bytes(t["ground"], t["ceiling"], None, *args)
    assert hashlib.sha256(built).hexdigest() == case["lga"]["built"]["sha256"]
    ev = lga_bytes(t["ground"], t["ceiling"], cost, *args)
    assert hashlib.sha256(ev).hexdigest() == case["lga"]["evaluated"]["sha256"]
    keep = oracle.simplify(t["ground"], cost)
    simp = lga_bytes(t["ground"][keep], t["ceiling"][keep], cost[keep], t["heights"][keep],
                     *args[1:])
    assert hashlib.sha256(simp).hexdigest() == case["lga"]["simplified"]["sha256"]


@pytest.mark.parametrize("name", ["ref_random_multilayer_s9", "ref_spiral_s3", "synth_cfg0"])
def test_oracle_planner_context_matches_reference(golden, name):
    from oracle.planner_ctx import planner_context
    case = golden["cases"][name]
    t = oracle.build(case_input(name, case), case["d_s"], case["r_g"])
    cost = oracle.evaluate(t["ground"], t["ceiling"], case["r_g"], TABLE_PARAMS)
    canon, cn = planner_context(t["ground"], cost)
    assert digest(canon) == case["planner"]["evaluated"]["canon_sha256"]
    assert digest(cn) == case["planner"]["evaluated"]["cn_sha256"]
    keep = case["keep"]
    canon, cn = planner_context(t["ground"][keep], cost[keep])
    assert digest(canon) == case["planner"]["simplified"]["canon_sha256"]
    assert digest(cn) == case["planner"]["simplified"]["cn_sha256"]

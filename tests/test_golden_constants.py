"""Pins the hyper-parameters the oracle and the product path default to against the values the paper
prints (tests/golden/paper_constants.json, each entry citing its PAPER.md line).  A mistyped threshold
or learning rate on either side fails here, independently of the parity tests (which compare the two
sides with the same arguments)."""
import inspect
import json
import math
import os

import pytest

from oracle import classify as OC, insert as OI, optim as OO, raster as OR, state as OS

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))


def g(key):
    return GOLD[key]["value"]


def defaults(fn):
    return {k: p.default for k, p in inspect.signature(fn).parameters.items() if p.default is not p.empty}


def test_delta_alpha_is_exp_minus_half():
    assert OR.DELTA_ALPHA == pytest.approx(g("delta_alpha"), rel=0, abs=1e-15)
    assert g("delta_alpha") == pytest.approx(math.exp(-0.5), rel=0, abs=1e-15)


def test_oracle_classify_thresholds():
    d = defaults(OC.classify)
    assert (d["delta_T"], d["delta_d"], d["delta_c"], d["ratio"]) == \
        (g("delta_T"), g("delta_d"), g("delta_c"), g("add_sample_ratio"))


def test_oracle_state_thresholds():
    fns = [f for _, f in inspect.getmembers(OS, inspect.isfunction) if "delta_eta" in defaults(f)]
    assert fns, "oracle/state.py exposes the state thresholds as defaults"
    for f in fns:
        d = defaults(f)
        assert d["delta_eta"] == g("delta_eta_replica")
        assert d["delta_c"] == g("delta_c") and d["delta_d"] == g("delta_d")


def test_oracle_insert_transparent_cap():
    assert defaults(OI.add_gaussians)["max_scale_transparent"] == g("transparent_max_scale_m")


def test_oracle_lr_vector_layout():
    lr = g("lr_replica")
    v = OO.lr_vector(16, lr["position"], lr["sh0"], g("lr_sh_rest_factor") * lr["sh0"], lr["scale"], lr["rotation"])
    assert len(v) == 3 + 3 + 4 + 3 + 45
    assert list(v[:3]) == [lr["position"]] * 3 and list(v[3:6]) == [lr["scale"]] * 3
    assert list(v[6:10]) == [lr["rotation"]] * 4 and list(v[10:13]) == [lr["sh0"]] * 3
    assert all(x == pytest.approx(0.05 * lr["sh0"]) for x in v[13:])


@pytest.mark.parametrize("preset,key", [("replica", "lr_replica"), ("scannetpp", "lr_replica"), ("tum", "lr_tum")])
def test_product_learning_rates(preset, key):
    from paper_2404_19706_b200 import mapping as M
    hp, lr = M.hparams(preset), g(key)
    assert (hp.lr_pos, hp.lr_sh0, hp.lr_scale, hp.lr_rot) == pytest.approx(
        (lr["position"], lr["sh0"], lr["scale"], lr["rotation"]), rel=1e-7)
    assert hp.lr_shrest == pytest.approx(g("lr_sh_rest_factor") * lr["sh0"], rel=1e-7)


def test_product_thresholds_and_weights():
    from paper_2404_19706_b200 import mapping as M
    a = M.add_params()
    assert (a.delta_T, a.delta_d, a.delta_c, a.sample_ratio) == pytest.approx(
        (g("delta_T"), g("delta_d"), g("delta_c"), g("add_sample_ratio")), rel=1e-7)
    s = M.state_params(0)
    assert s.delta_eta == g("delta_eta_replica")
    assert (s.delta_c, s.delta_d) == pytest.approx((g("delta_c"), g("delta_d")), rel=1e-7)
    w = defaults(M.MappingEngine.__init__)["weights"]
    assert tuple(w) == (g("w_c"), g("w_d"), g("w_reg"))
    gs = defaults(M.MappingEngine.global_step)
    assert (gs["ratio"], gs["lr_scale"]) == (g("global_top_error_ratio"), g("global_lr_factor"))

"""Config front end (paper_2202_06111_b200.config) against the reference's
cg/config.py, pinned by tests/golden/config.json (make_golden.py gen_config:
the reference's own resolve_config / parse_config_text / render_config on
valid and invalid inputs).  Mirrors /root/reference/pkg/tests/test_cli.py
TestConfig."""
import json
import os
from pathlib import Path

import numpy as np
import pytest

from paper_2202_06111_b200.config import (WORKERS_ENV_VAR, ConfigError, parse_config_text,
                                          render_config, resolve_config)

GOLDEN = json.loads((Path(__file__).parent / "golden" / "config.json").read_text())


def _summary(rc):
    m = rc.model
    return {"model": m.name, "n": m.n, "m": m.m,
            "X": [list(map(float, m.X.lo)), list(map(float, m.X.hi))],
            "U": [list(map(float, m.U.lo)), list(map(float, m.U.hi))],
            "iterations": rc.iterations, "min_diameter": rc.min_diameter,
            "mode": rc.adaptive.mode, "N": rc.adaptive.n_neighbors, "delta": rc.adaptive.delta,
            "include_face_points": rc.adaptive.include_face_points,
            "samples_per_dim": rc.image.samples_per_dim, "bloat": rc.image.bloat,
            "batch_size": rc.plan.batch_size, "workers": rc.plan.workers,
            "input_counts": rc.input_counts if isinstance(rc.input_counts, int)
            else list(rc.input_counts),
            "strict_largest_scc": rc.strict_largest_scc}


def _resolve(case, monkeypatch):
    monkeypatch.delenv(WORKERS_ENV_VAR, raising=False)
    if case["env_workers"] is not None:
        monkeypatch.setenv(WORKERS_ENV_VAR, case["env_workers"])
    return resolve_config(case["file"], case["overrides"])


@pytest.mark.parametrize("i", range(len(GOLDEN["cases"])))
def test_resolve_matches_reference(i, monkeypatch):
    case = GOLDEN["cases"][i]
    if "error_key" in case:
        with pytest.raises(ConfigError) as err:
            _resolve(case, monkeypatch)
        assert err.value.key == case["error_key"]
        assert str(err.value) == case["error"]
        return
    r = _resolve(case, monkeypatch)
    assert r.effective == case["effective"]
    assert render_config(r.effective) == case["rendered"]
    assert parse_config_text(render_config(r.effective)) == r.effective
    assert _summary(r.run_config) == case["run_config"]


@pytest.mark.parametrize("i", range(len(GOLDEN["texts"])))
def test_parse_matches_reference(i):
    t = GOLDEN["texts"][i]
    if "error_key" in t:
        with pytest.raises(ConfigError) as err:
            parse_config_text(t["text"])
        assert err.value.key == t["error_key"] and str(err.value) == t["error"]
    else:
        assert parse_config_text(t["text"]) == t["values"]


def test_reference_test_cli_config_behaviours(monkeypatch):
    # tests/test_cli.py:21-65 of the reference, restated
    values = parse_config_text("iterations = 12\nmodel = linear\nlinear.a = 2.0\n")
    assert values == {"iterations": "12", "model": "linear", "linear.a": "2.0"}
    assert parse_config_text(render_config(values)) == values
    assert parse_config_text("# a comment\n\nmode = adaptive  # trailing\n") == {"mode": "adaptive"}
    for bad, key in (({"cell_count": "4"}, "cell_count"), ({"iterations": "many"}, "iterations"),
                     ({"model": "cstr", "linear.a": "2"}, "linear.a")):
        with pytest.raises(ConfigError) as err:
            resolve_config(bad)
        assert key in str(err.value)
    assert resolve_config({"iterations": "5"}, {"iterations": "7"}).run_config.iterations == 7
    monkeypatch.setenv(WORKERS_ENV_VAR, "3")
    r = resolve_config({}, {"workers": "1"})
    assert r.run_config.plan.workers == 3 and r.effective["workers"] == "3"
    monkeypatch.delenv(WORKERS_ENV_VAR)
    rc = resolve_config({}).run_config
    assert rc.model.name == "cstr" and rc.iterations == 20 and rc.adaptive.n_neighbors == 3
    assert rc.image.samples_per_dim == 3 and rc.image.bloat == 0.1
    assert rc.plan.batch_size == 1024


@pytest.mark.gpu
def test_resolved_models_step_like_reference(monkeypatch):
    """The resolved model's step (libgis gis_map_points) on the recorded
    points equals the reference model's, within the 1e-12 contract."""
    for case in GOLDEN["cases"]:
        if "error_key" in case:
            continue
        model = _resolve(case, monkeypatch).run_config.model
        got = np.asarray(model.map_points(np.asarray(case["x"]), np.asarray(case["u"])))
        want = np.asarray(case["step"])
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-300)

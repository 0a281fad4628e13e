"""Cost-model JSON boundary (moesim/simulator.py:64-92): the file we write
must load through CostModel.from_json_obj; measured fields on a B200."""

import json

import pytest

from paper_2501_10375_b200 import costmodel
from paper_2501_10375_b200.errors import ConfigError, MoesimError

# moesim/simulator.py:49-55 defaults, a valid override set
DEFAULTS = {"t_nonmoe_fast": 0.24, "t_expert_fast": 0.50, "t_expert_slow": 3.20,
            "t_gate": 0.01, "t_migrate_expert": 39.87, "t_activation_xfer": 0.02,
            "slow_parallelism": 1}


def test_fields_match_reference_order():
    assert costmodel.FIELDS == tuple(DEFAULTS)


def test_round_trip_drops_detail(tmp_path):
    obj = dict(DEFAULTS, _detail={"gpu": "x"})
    p = tmp_path / "c.json"
    costmodel.save(obj, p)
    assert json.loads(p.read_text()) == DEFAULTS
    assert costmodel.load(p) == DEFAULTS


def test_partial_override_is_valid():
    assert costmodel.validate({"t_gate": 0.0}) == {"t_gate": 0.0}


@pytest.mark.parametrize("bad", [{"t_gate": -1e-9}, {"t_expert_slow": float("nan")},
                                 {"slow_parallelism": 0}, {"slow_parallelism": 1.5},
                                 {"t_fast": 1.0}])
def test_rejects_what_the_reference_rejects(bad):
    with pytest.raises(ConfigError):
        costmodel.validate(bad)
    assert issubclass(ConfigError, MoesimError)


@pytest.mark.gpu
def test_measure_small_shape(tmp_path):
    res = costmodel.measure(d=512, ffn=1024, ctx=64, reps=5, host_reps=2)
    for f in costmodel.FIELDS[:-1]:
        assert res[f] > 0, f
    assert res["slow_parallelism"] == 1
    # the layer streams k experts: one expert costs less than the whole layer
    assert res["t_expert_fast"] < res["_detail"]["decode_layer_ms"]
    p = tmp_path / "c.json"
    costmodel.save(res, p)
    assert set(costmodel.load(p)) == set(costmodel.FIELDS)

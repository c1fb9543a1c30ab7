"""Instance generator / JSON format parity with the reference (model.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1704_05132_b200.model import (GeneratorConfig, Instance, InstanceFormatError,
                                         generate_instance, parse_instance,
                                         serialize_instance, validate_instance)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


with open(os.path.join(GOLDEN, "instances.json")) as f:
    _INSTANCES = json.load(f)


@pytest.mark.parametrize("entry", _INSTANCES, ids=lambda e: str(e["config"]))
def test_generator_bit_identical_to_reference(entry):
    cfg = dict(entry["config"])
    if cfg["products"] * cfg["periods"] > 2_000_000:
        pytest.skip("large configs covered by the GPU bench path")
    inst = generate_instance(GeneratorConfig(**cfg))
    names = ("demand", "returns", "setup_cost_m", "setup_cost_r", "holding_cost_m",
             "holding_cost_r", "unit_cost_m", "unit_cost_r")
    for name, arr in zip(names, inst.arrays()):
        assert _sha(arr) == entry["sha256"][name], name


def test_json_round_trip_and_errors():
    inst = generate_instance(GeneratorConfig(products=3, periods=4, seed=1))
    assert parse_instance(serialize_instance(inst)) == inst
    with pytest.raises(InstanceFormatError):
        parse_instance("{")
    with pytest.raises(InstanceFormatError):
        parse_instance(json.dumps({"products": 1}))
    bad = json.loads(serialize_instance(inst))
    bad["demand"][0][0] = -1
    with pytest.raises(InstanceFormatError):
        parse_instance(json.dumps(bad))
    bad = json.loads(serialize_instance(inst))
    bad["extra"] = 1
    with pytest.raises(InstanceFormatError):
        parse_instance(json.dumps(bad))


def test_validate_and_config_errors():
    inst = Instance(1, 2, [[1, -1]], [[0, 0]], [1], [1], [1], [1])
    assert validate_instance(inst) == ["demand contains negative entries"]
    with pytest.raises(ValueError):
        GeneratorConfig(products=0, periods=1)
    with pytest.raises(ValueError):
        GeneratorConfig(products=1, periods=1, return_ratio=1.5)
    with pytest.raises(ValueError):
        GeneratorConfig(products=1, periods=1, setup_cost_range=(5, 1))

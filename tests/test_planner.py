"""The native planner (C ABI of libpipeplan_b200.so) is bit-exact with the
reference: golden fixtures from the compiled reference, the reference's own
partition tests (proj/tests/test_partition.cpp:41-219) restated, and the
oracle on random chains.  CPU only (no CUDA call)."""
import random

import numpy as np
import pytest

from _util import golden, oracle
from paper_2207_11019_b200 import api
from paper_2207_11019_b200.api import BoundaryKind, LayerSpec, ModelGraph, PipeplanError  # noqa: F401


def test_split_layer_golden():
    for e in golden()["split_layer"]:
        if "error" in e:
            with pytest.raises(PipeplanError) as ei:
                api.split_layer((3, e["fan_out"]), e["n"], e["replicate"])
            assert str(ei.value) == e["error"]
        else:
            got = api.split_layer((3, e["fan_out"]), e["n"], e["replicate"])
            assert [[s.lo, s.hi, s.replicated] for s in got] == e["shards"]


def test_split_microbatches_golden():
    for e in golden()["split_microbatches"]:
        if "error" in e:
            with pytest.raises((PipeplanError, ValueError)) as ei:
                api.split_microbatches(e["b"], e["m"])
            assert str(ei.value) == e["error"]
        else:
            assert api.split_microbatches(e["b"], e["m"]) == e["sizes"]


def test_build_plan_golden():
    for e in golden()["build_plan"]:
        if "error" in e:
            with pytest.raises((PipeplanError, ValueError)) as ei:
                api.build_plan(e["dims"], e["n"], e["Z"], e["replicate"])
            assert str(ei.value) == e["error"]
            continue
        p = api.build_plan(e["dims"], e["n"], e["Z"], e["replicate"])
        assert p.to_flat().tolist() == e["plan"]
        api.validate_plan(p, e["dims"])
        if "merged_1_2" in e:
            assert api.merge_submodules(p, [1, 2]).to_flat().tolist() == e["merged_1_2"]
            assert api.merge_all(p).to_flat().tolist() == e["merged_all"]


def test_build_staged_plan_golden():
    for e in golden()["build_staged_plan"]:
        assert api.build_staged_plan(e["dims"], e["groups"]).to_flat().tolist() == e["plan"]


# ---- restatement of proj/tests/test_partition.cpp ----

def uniform(L, width):
    return ModelGraph([LayerSpec(i + 1, width, width) for i in range(L)])


def test_split_layer_balances_largest_remainder_first():  # :41-60
    s = api.split_layer(LayerSpec(1, 4, 8), 2)
    assert [(x.lo, x.hi) for x in s] == [(0, 4), (4, 8)]
    s = api.split_layer(LayerSpec(1, 4, 7), 2)
    assert [(x.lo, x.hi) for x in s] == [(0, 4), (4, 7)]
    s = api.split_layer(LayerSpec(1, 4, 8), 1)
    assert [(x.lo, x.hi) for x in s] == [(0, 8)]


def test_split_layer_rejects_narrow():  # :62-73
    with pytest.raises(PipeplanError, match="too narrow"):
        api.split_layer(LayerSpec(1, 4, 2), 3)
    s = api.split_layer(LayerSpec(1, 4, 2), 3, True)
    assert all(x.replicated and x.lo == 0 and x.hi == 2 for x in s) and len(s) == 3


def test_split_tiling_property():  # :75-95 (same generator family, own seed)
    rng = random.Random(42)
    for _ in range(200):
        fo, n = 1 + rng.randrange(32), 1 + rng.randrange(8)
        if fo < n:
            continue
        s = api.split_layer(LayerSpec(1, 3, fo), n)
        lo = 0
        for x in s:
            assert x.lo == lo
            lo = x.hi
        assert lo == fo
        u = [x.units() for x in s]
        assert max(u) - min(u) <= 1


def test_build_plan_two_balanced_spans():  # :97-108
    p = api.build_plan(uniform(4, 8), 2, 2)
    assert [(sm.first_layer, sm.last_layer) for sm in p.submodules] == [(1, 2), (3, 4)]
    assert p.boundaries == [BoundaryKind.concat_repartition]


def test_build_plan_singletons_and_z_bounds():  # :110-119
    p = api.build_plan(uniform(3, 6), 2, 3)
    assert p.num_submodules() == 3 and len(p.boundaries) == 2
    assert all(sm.num_layers() == 1 for sm in p.submodules)
    with pytest.raises(PipeplanError, match="Z exceeds layer count"):
        api.build_plan(uniform(2, 6), 2, 3)


def test_build_plan_deterministic():  # :121-126
    a = api.build_plan(uniform(5, 12), 3, 2)
    b = api.build_plan(uniform(5, 12), 3, 2)
    assert a.to_flat().tolist() == b.to_flat().tolist()


def test_merge_semantics():  # :128-153
    p = api.build_plan(uniform(3, 6), 2, 3)
    m = api.merge_submodules(p, [1, 2])
    assert m.boundaries == [BoundaryKind.direct, BoundaryKind.concat_repartition]
    assert m.num_submodules() == 3
    assert [s.to_flat().tolist() for s in [p]] != [m.to_flat().tolist()]
    assert m.provenance == ["merge[1..2]"]
    with pytest.raises(PipeplanError, match="contiguous"):
        api.merge_submodules(p, [1, 3])
    with pytest.raises(PipeplanError, match="out of range"):
        api.merge_submodules(p, [2, 4])
    assert api.merge_all(p).boundaries == [BoundaryKind.direct] * 2


def test_validate_plan_errors():  # :213-219 and partition.cpp:232-294
    p = api.build_plan([4, 8, 8], 2, 1)
    api.validate_plan(p, [4, 8, 8])
    with pytest.raises(PipeplanError, match="absent from the cluster"):
        api.validate_plan(p, [4, 8, 8], cluster_devices=1)
    with pytest.raises(PipeplanError, match="tile"):
        api.validate_plan(p, [4, 8, 9])


def test_planner_matches_oracle_random():
    O = oracle()
    rng = random.Random(7)
    for _ in range(300):
        L = rng.randint(1, 6)
        dims = [rng.randint(1, 40) for _ in range(L + 1)]
        n, Z, rep = rng.randint(1, 8), rng.randint(1, L), rng.random() < 0.5
        try:
            ref = O.build_plan(dims, n, Z, rep).tolist()
        except Exception as e:  # noqa: BLE001
            with pytest.raises((PipeplanError, ValueError)) as ei:
                api.build_plan(dims, n, Z, rep)
            assert str(ei.value) == str(e)
            continue
        assert api.build_plan(dims, n, Z, rep).to_flat().tolist() == ref


def test_serialize_plan_byte_identical_to_reference():
    """partition.cpp:303-331: the same JSON text the reference writes."""
    for e in golden()["serialize_plan"]:
        p = api.PartitionPlan.from_flat(e["plan"], e["provenance"])
        assert api.serialize_plan(p) == e["json"]


def test_parse_plan_round_trip_and_errors():
    for e in golden()["serialize_plan"]:
        p = api.parse_plan(e["json"])
        assert p.to_flat().tolist() == e["plan"]
        assert p.provenance == e["provenance"]
    for e in golden()["parse_plan"]:
        if "error" in e:
            with pytest.raises(PipeplanError) as ei:
                api.parse_plan(e["text"])
            assert str(ei.value) == e["error"]
        else:
            assert api.parse_plan(e["text"]).to_flat().tolist() == e["plan"]
    with pytest.raises(PipeplanError, match="plan parse error"):
        api.parse_plan("{not json")
    with pytest.raises(PipeplanError, match="key 'n' not found"):
        api.parse_plan('{"submodules": [], "boundaries": []}')

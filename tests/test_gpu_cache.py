"""Measurement caches on the device: validation against the device-enumerated
space (MeasurementCache::validate, cache.hpp:74-108) and simulation-mode
replay reproducing the unmodified reference's trajectory on the same cache."""
import pathlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = pathlib.Path(__file__).parent / "golden"


def test_replay_reproduces_reference_trajectory(gt, tmp_path):
    c = gt.MeasurementCache.load_json(GOLDEN / "cache_rr13.json")  # random-rough 13x13 s17 inv 0.3
    c.save_binary(tmp_path / "rr13.bin")
    es, values = gt.MeasurementCache.load(tmp_path / "rr13.bin").replay()
    t = np.load(GOLDEN / "traj_rr13_ei.npz")  # same space, reference run_bo bo-ei seed 1
    np.testing.assert_array_equal(es.ids, t["ids"])
    assert es.coords.tobytes() == np.ascontiguousarray(t["coords"]).tobytes()
    run = gt.run_bo(es, es.ids, gt.StrategyConfig(id=gt.StrategyId.bo_ei, seed=1, budget=70, n_init=12),
                    values=values)
    np.testing.assert_array_equal(run.positions, t["traj_pos"])


def test_validation_errors(gt):
    c = gt.MeasurementCache.load_json(GOLDEN / "cache_rr4d.json")
    c.validate()
    short = gt.MeasurementCache(c.kernel_name, c.params, c.restrictions, c.ids[:-1], c.values[:-1], c.reasons[:-1])
    with pytest.raises(gt.CacheError, match="entries but the space has"):
        short.validate()
    neg = gt.MeasurementCache(c.kernel_name, c.params, c.restrictions, c.ids, -c.values, c.reasons)
    with pytest.raises(gt.CacheError, match="non-positive value"):
        neg.validate()
    c.true_minimum = 0.5
    with pytest.raises(gt.CacheError, match="states minimum"):
        c.validate()


def test_load_validates_like_the_reference(gt, tmp_path):
    """MeasurementCache::load ends with validate() (cache.hpp:236): a cache
    missing one configuration is rejected at load time."""
    import json
    doc = json.loads((GOLDEN / "cache_rr4d.json").read_text())
    gone = doc["entries"].pop(4)
    (tmp_path / "short.json").write_text(json.dumps({k: v for k, v in doc.items() if k != "checksum"}))
    with pytest.raises(gt.CacheError, match="entries but the space has"):
        gt.MeasurementCache.load(tmp_path / "short.json")
    # same count, one configuration replaced by an index outside the space
    doc["entries"].append({"index": 10 ** 12, "value": 1.0})
    doc.pop("checksum")
    (tmp_path / "m.json").write_text(json.dumps(doc))
    with pytest.raises(gt.CacheError, match=f"missing an entry for configuration {gone['index']}"):
        gt.MeasurementCache.load(tmp_path / "m.json")
    assert len(gt.MeasurementCache.load(GOLDEN / "cache_rr4d.json").ids) == len(doc["entries"])

"""Measurement caches without a GPU: the reference's JSON caches
(tests/golden/cache_*.json, written by MeasurementCache::save of the
unmodified reference via oracle/_ref/ref_tool cachegen) load with the
reference's FNV-1a checksum (cache.hpp:55-70, native gtc_cache_checksum),
and the binary format round-trips them exactly; corruption is detected."""
import json
import pathlib

import numpy as np
import pytest

GOLDEN = pathlib.Path(__file__).parent / "golden"
CACHES = ["cache_rr13", "cache_rosen", "cache_rr4d"]


@pytest.mark.parametrize("name", CACHES)
def test_reference_json_checksum(gt, name):
    path = GOLDEN / f"{name}.json"
    c = gt.MeasurementCache.load_json(path, validate=False)
    doc = json.loads(path.read_text())
    assert "fnv1a64:%016x" % c.checksum() == doc["checksum"]
    assert len(c.ids) == len(doc["entries"])
    assert c.invalid_count() == sum("invalid" in e for e in doc["entries"])
    if "true_minimum" in doc:
        assert c.min_valid_value() == doc["true_minimum"]


@pytest.mark.parametrize("name", CACHES)
def test_binary_and_json_round_trips(gt, name, tmp_path):
    c = gt.MeasurementCache.load_json(GOLDEN / f"{name}.json", validate=False)
    c.save_binary(tmp_path / "c.bin")
    b = gt.MeasurementCache.load(tmp_path / "c.bin", validate=False)
    np.testing.assert_array_equal(b.ids, c.ids)
    np.testing.assert_array_equal(b.reasons, c.reasons)
    assert b.values.tobytes() == c.values.tobytes()
    assert b.checksum() == c.checksum() and b.kernel_name == c.kernel_name
    assert [p.values for p in b.params] == [p.values for p in c.params]
    assert (tmp_path / "c.bin").stat().st_size < (GOLDEN / f"{name}.json").stat().st_size / 4
    c.save_json(tmp_path / "c.json")
    j = gt.MeasurementCache.load(tmp_path / "c.json", validate=False)
    assert j.checksum() == c.checksum()
    np.testing.assert_array_equal(j.ids, c.ids)


def test_corruption_is_detected(gt, tmp_path):
    c = gt.MeasurementCache.load_json(GOLDEN / "cache_rr4d.json", validate=False)
    c.save_binary(tmp_path / "c.bin")
    raw = bytearray((tmp_path / "c.bin").read_bytes())
    raw[-len(c.ids) - 3] ^= 0x40  # a value byte
    (tmp_path / "bad.bin").write_bytes(bytes(raw))
    with pytest.raises(gt.CacheError, match="checksum mismatch"):
        gt.MeasurementCache.load(tmp_path / "bad.bin", validate=False)
    (tmp_path / "short.bin").write_bytes(bytes(raw[:-5]))
    with pytest.raises(gt.CacheError, match="truncated"):
        gt.MeasurementCache.load(tmp_path / "short.bin", validate=False)
    doc = json.loads((GOLDEN / "cache_rr4d.json").read_text())
    doc["schema_version"] = 2
    (tmp_path / "v2.json").write_text(json.dumps(doc))
    with pytest.raises(gt.CacheError, match="unsupported cache schema version"):
        gt.MeasurementCache.load(tmp_path / "v2.json", validate=False)


def test_entry_checks_of_the_reference_loader(gt, tmp_path):
    """MeasurementCache::load's per-entry checks (cache.hpp:200-225), in file
    order: the embedded config tuple against its index, then duplicates."""
    doc = json.loads((GOLDEN / "cache_rr4d.json").read_text())
    e = doc["entries"]
    assert all("config" in x for x in e)

    def load(d, name):
        (tmp_path / name).write_text(json.dumps(d))
        return gt.MeasurementCache.load_json(tmp_path / name, validate=False)

    bad = json.loads(json.dumps(doc))
    bad["entries"][3]["config"] = bad["entries"][3]["config"][:-1]
    with pytest.raises(gt.CacheError, match=f"entry {e[3]['index']} config tuple has wrong arity"):
        load(bad, "arity.json")
    bad = json.loads(json.dumps(doc))
    bad["entries"][5]["config"] = bad["entries"][6]["config"]
    with pytest.raises(gt.CacheError, match=f"entry {e[5]['index']} config tuple does not match its index"):
        load(bad, "tuple.json")
    bad = json.loads(json.dumps(doc))
    bad["entries"].append(dict(bad["entries"][2]))
    with pytest.raises(gt.CacheError, match=f"duplicate entry for configuration {e[2]['index']}"):
        load(bad, "dup.json")
    bad = json.loads(json.dumps(doc))
    bad["restrictions"] = ["x0 <"]
    with pytest.raises(gt.ParseError):
        load(bad, "restr.json")
    ok = load(doc, "ok.json")
    assert ok.config_at(int(e[7]["index"])) == e[7]["config"]

"""Restriction language and search-space validation against the UNMODIFIED
reference, without a GPU: parse outcomes, ParseError messages and positions
(tests/golden/restrictions.json: the reference KATs of test_restriction.cpp
plus a seeded fuzz set, all produced by oracle/_ref/ref_tool) and SearchSpace
construction errors (tests/golden/enum_errors.json).  Parsing and validation
happen in the C ABI layer before any device work."""
import json
import pathlib

import pytest

GOLDEN = pathlib.Path(__file__).parent / "golden"


def defs(gt, spec):
    return [gt.ParameterDef(p["name"], p["values"], gt.ParamKind[p["kind"]]) for p in spec]


def test_restriction_parse_matches_reference(gt):
    data = json.loads((GOLDEN / "restrictions.json").read_text())
    params = defs(gt, data["params"])
    n_ok = 0
    for case in data["cases"]:
        text = case["text"]
        if case["ok"]:
            assert gt.parse_restriction(text, params) == text
            n_ok += 1
        else:
            with pytest.raises(gt.ParseError) as e:
                gt.parse_restriction(text, params)
            assert str(e.value) == case["message"], text
            assert e.value.position == case["position"], text
    assert n_ok > 250 and len(data["cases"]) - n_ok > 100


@pytest.mark.parametrize("name", ["dup_param", "dup_value", "dup_zero", "dup_bool", "dup_string", "bad_name",
                                  "no_values", "parse_first", "too_big"])
def test_search_space_errors_match_reference(gt, name):
    case = json.loads((GOLDEN / "enum_errors.json").read_text())[name]
    spec, want = case["spec"], case["result"]
    space = gt.SearchSpace(defs(gt, spec["params"]), spec.get("restrictions", []))
    exc = gt.ParseError if want["error"] == "parse" else gt.Error
    with pytest.raises(exc) as e:
        space.enumerate()
    assert str(e.value) == want["message"]
    if want["error"] == "parse":
        assert e.value.position == want["position"]

"""The oracle's full-size exact-integer results (tests/golden/oracle_fullsize.json, written by
tools/make_golden.py calling only oracle/ and synthgen/) against SURVEY.md §8 c7's independently
computed checksums and corners (tests/golden/survey_c7.json).  CPU only: reads two JSON files.
A mismatch means the oracle (or the generator) disagrees with an independent implementation at
the configs' full shapes — the values the GPU tests then hold the CUDA path to."""
import json
import os

import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLDEN, "oracle_fullsize.json")) as f:
    ORACLE = json.load(f)
with open(os.path.join(GOLDEN, "survey_c7.json")) as f:
    SURVEY = json.load(f)


@pytest.mark.parametrize("key", ["C1x", "C2x", "C3", "C4x3", "C4x9", "C5x"])
def test_oracle_fullsize_matches_survey_c7(key):
    if key not in ORACLE:
        pytest.skip(f"{key}: oracle golden not generated (tools/make_golden.py --only {key})")
    o, s = ORACLE[key], SURVEY[key]
    assert int(o["checksum"], 16) == int(s["checksum"], 16), key
    assert o["C00"] == s["C00"], key
    if "Clast_last" in s:
        assert o["Clast_last"] == s["Clast_last"], key
    if "zeros" in s:
        assert o["zeros"] == s["zeros"], key

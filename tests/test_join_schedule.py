"""Join schedules (CPU): psg_join_schedule reproduces the reference's make_plan
(/root/reference/proj/src/join.cpp:55-134) step for step - phase, stream, wave - for all four
variants over stream counts and wave counts, pinned by tests/golden/join.json (made by
tests/golden/make_golden_join.py from the reference itself)."""
import json
import os

import pytest

import paper_2512_02862_b200 as psg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "join.json")))


@pytest.mark.parametrize("case", GOLD["schedules"], ids=lambda c: "%s-s%d-%dx%d" % (c["variant"], c["streams"], c["left"], c["right"]))
def test_schedule_matches_reference(case):
    got = psg.join_schedule(case["variant"], case["streams"], case["left"], case["right"])
    assert got == case["steps"]


def test_deferred_probe_lands_after_the_next_shuffle():
    """The property the deferred variant exists for: every probe of wave w (but the trailing
    ones) is issued after the shuffle of wave w + k on the same stream."""
    k = 2
    steps = psg.join_schedule("deferred", k, 3, 7)
    pos = {(ph, w): i for i, (ph, _s, w) in enumerate(steps)}
    for w in range(7 - k):
        assert pos[(9, w)] > pos[(8, w + k - 1)]
        assert pos[(9, w)] < pos[(6, w + k)]


def test_bad_variant_is_invalid_input():
    with pytest.raises(psg.PsgError) as e:
        psg.join_schedule(7, 1, 1, 1)
    assert e.value.kind == "InvalidInput"

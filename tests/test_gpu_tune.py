"""tileqr_tune replayed through the oracle's tuner.

The library times Step 1 and Step 2 on the GPU and writes every sample it
decided on into its JSON report (exact values, %.17g).  Feeding those same
samples through oracle/tuner.py -- Property 1 with the report's tie width,
the upper hull, Heuristic 0/1/2, Property 3 between the
rungs of the ladder -- must reproduce the library's
candidate set, the survivors timed at every rung and the final pick.
"""
import json

import pytest

from oracle import tuner

pytestmark = pytest.mark.gpu

NB_GRID = (64, 96, 128, 160, 192, 224, 256)


@pytest.fixture(scope="module")
def tq():
    from paper_1102_5328_b200 import tileqr
    return tileqr


def replay(report, heuristic, payg, nb, ib):
    s1 = [(p["nb"], p["ib"], p["gflops"]) for p in report["step1"]]
    grid = sorted((b, i) for b in NB_GRID for i in range(8, b + 1) if b % i == 0)
    assert sorted((b, i) for b, i, _ in s1) == grid                      # every (NB, IB >= 8) timed once
    assert all(g > 0 for _, _, g in s1)
    cand = tuner.preselect(s1, heuristic, 8, report["tie_rel"])
    assert sorted((b, i) for b, i, _ in cand) == sorted((p["nb"], p["ib"]) for p in report["candidates"])
    ladder = sorted({p["n"] for p in report["step2"]})
    assert ladder[-1] == report["N"]
    alive = {(b, i) for b, i, _ in cand}
    rung = []
    for n in ladder:
        rung = [(p["nb"], p["ib"], p["gflops"]) for p in report["step2"] if p["n"] == n]
        assert {(b, i) for b, i, _ in rung} == alive, n                   # survivors of the previous rung
        if payg:
            alive = {(b, i) for b, i, _ in tuner.payg_prune(rung)}
    best = rung[0]
    for r in rung:
        if r[2] > best[2]:
            best = r
    assert (nb, ib) == best[:2] == (report["best"]["nb"], report["best"]["ib"])


@pytest.mark.parametrize("heuristic,payg", [(2, True), (1, False), (0, True)])
def test_tune_replays_through_oracle(tq, tmp_path, monkeypatch, heuristic, payg):
    monkeypatch.setenv("TILEQR_TUNE_BATCH", "96")
    monkeypatch.setenv("TILEQR_TUNE_REPS", "3")
    path = tmp_path / "tune.json"
    nb, ib = tq.tune(1024, 1024, 1, heuristic, payg, str(path))
    report = json.load(open(path))
    assert report["heuristic"] == heuristic and report["payg"] == int(payg)
    replay(report, heuristic, payg, nb, ib)
    tq.finalize()

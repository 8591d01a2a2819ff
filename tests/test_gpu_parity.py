"""GPU vs CPU oracle on seeded synthetic traces of every SURVEY.md §8(d) configuration shape.

Bit-exact comparison of the TallyReport, IntervalStats, the ordered orphan
list and the timeline JSON bytes.  Sizes are chosen so the oracle finishes in seconds; the full-size
workloads are exercised by bench.py with size-independent checks."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2504_03683_b200.engine import Engine

    eng = Engine(device=0)
    yield eng
    eng.close()


def _cmp(engine, wl, timeline=True):
    """Report, stats, orphans and (tally + timeline run) the timeline JSON bytes."""
    from oracle import oracle
    from paper_2504_03683_b200 import synth

    raws = synth.generate(wl)
    infos = [r.info for r in raws]
    got = engine.run(raws, wl.registry, infos, want_timeline=timeline)
    want = oracle.run(raws, wl.registry, infos, want_timeline=timeline)
    assert (got.error is None) == (want.error is None), (got.error, want.error)
    if want.error is not None:
        assert type(got.error) is type(want.error) and str(got.error) == str(want.error)
        return got
    assert got.stats == want.stats
    assert got.report == want.report
    assert got.orphans == want.orphans
    if timeline:
        assert got.timeline == want.timeline.encode()
    return got


@pytest.mark.parametrize("name,scale", [("c1", 0.05), ("c2", 0.01), ("c3", 0.001), ("c4", 0.005), ("c5", 0.005)])
def test_configs_match_oracle(engine, name, scale):
    from paper_2504_03683_b200 import synth

    got = _cmp(engine, synth.config(name, scale))
    assert got.stats["events_in"] > 0


@pytest.mark.parametrize("seed", range(6))
def test_adversarial_structure_matches_oracle(engine, seed):
    """Orphans, typed mismatches, unclosed calls, annotations, equal timestamps, deep stacks."""
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    params = dict(orphan_p=0.01 * seed, mismatch_p=0.02 * (seed % 3), meta_p=0.03, close_at_end=seed % 2,
                  max_depth=[4, 8, 64, 300, 2, 16][seed], push_p=[0.5, 0.6, 0.7, 0.9, 0.5, 0.55][seed],
                  gap_lo=0, gap_hi=[3, 600, 1, 50, 0, 5][seed], prof_p=0.3)
    streams = [synth.StreamSpec(f"h{i % 3}", P + 100 * (i % 4), P + 100 * (i % 4) + i, 3000 + 997 * i,
                                9000 + 31 * seed + i) for i in range(12)]
    wl = synth.Workload(f"adv{seed}", synth.ze_registry(), streams, params, kernel_names=synth.kernel_pool(30))
    _cmp(engine, wl)


def test_single_huge_stream_matches_oracle(engine):
    """One stream spanning thousands of tiles: look-back chains over a single stream."""
    from paper_2504_03683_b200 import synth

    wl = synth.Workload("big1", synth.ze_registry(), [synth.StreamSpec("s", 1, 1, 400_000, 77)],
                        {"max_depth": 12, "push_p": 0.55, "mismatch_p": 0.001, "close_at_end": 0})
    _cmp(engine, wl)


def test_timeline_many_runs_and_empty_streams(engine):
    """2,100 streams (over 1,024 merge pairs in the first pass), every seventh empty, unclosed
    calls (truncated spans sorted among compose's messages)."""
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    streams = [synth.StreamSpec(f"h{i % 5}", P + 100 * (i % 9), P + 100 * (i % 9) + i, 0 if i % 7 == 3 else 20 + i % 61,
                                5000 + i) for i in range(2100)]
    wl = synth.Workload("many", synth.ze_registry(), streams, {"close_at_end": 0, "prof_p": 0.3},
                        kernel_names=synth.kernel_pool(40))
    _cmp(engine, wl)


def test_timeline_record_region_over_1024_tiles(engine):
    """Over 2M record slots: the tile-count scan of the run compaction spans several CTA rounds."""
    from paper_2504_03683_b200 import synth

    _cmp(engine, synth.config("c2", 0.022))  # 2.2M records: 1,074 tiles

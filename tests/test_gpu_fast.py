"""The single-pass range path (csrc/fast.cuh) against the CPU oracle.

Tally-only runs take the single pass; it must be bit-exact with the oracle on
every configuration shape, at the default range size and at small range sizes
that put many speculative range starts inside records.  Traces the single pass
cannot vouch for (errors) must fall back to the exact path and still match."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2504_03683_b200.engine import Engine

    eng = Engine(device=0)
    yield eng
    eng.close()


def _run(engine, wl, range_bytes=0, path=0):
    from oracle import oracle
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.engine import OPT_PATH, OPT_RANGE_BYTES

    raws = synth.generate(wl)
    infos = [r.info for r in raws]
    engine.set_option(OPT_PATH, path)
    engine.set_option(OPT_RANGE_BYTES, range_bytes)
    try:
        got = engine.run(raws, wl.registry, infos)
    finally:
        engine.set_option(OPT_PATH, 0)
        engine.set_option(OPT_RANGE_BYTES, 0)
    want = oracle.run(raws, wl.registry, infos)
    assert (got.error is None) == (want.error is None), (got.error, want.error)
    if want.error is None:
        assert got.stats == want.stats
        assert got.report == want.report
        assert got.orphans == want.orphans
    else:
        assert type(got.error) is type(want.error) and str(got.error) == str(want.error)
    return got


@pytest.mark.parametrize("range_bytes", [0, 512, 1008, 4096])
@pytest.mark.parametrize("name,scale", [("c1", 0.02), ("c2", 0.004), ("c3", 0.0005), ("c4", 0.003), ("c5", 0.003)])
def test_single_pass_matches_oracle(engine, name, scale, range_bytes):
    from paper_2504_03683_b200 import synth

    _run(engine, synth.config(name, scale), range_bytes, path=2)
    assert engine.last_path()[0] == 1


@pytest.mark.parametrize("range_bytes", [512, 1008])
@pytest.mark.parametrize("name,scale", [("c2", 0.03), ("c5", 0.03)])
def test_several_ranges_per_lane(engine, name, scale, range_bytes):
    """More ranges than lanes (148 SMs x 12 warps x 32): lanes walk several ranges one after the
    other, and the ring of the next range must not count the previous range's fills as its own.
    A forced range size disables the retry with shifted cut points, so a speculated range start
    that self-synchronises inside a device record (c5 at 1008 B) falls back to the exact path."""
    from paper_2504_03683_b200 import synth

    wl = synth.config(name, scale)  # ~96 MB (c2), ~100 MB (c5): 95k-200k ranges over 56832 lanes
    _run(engine, wl, range_bytes)
    if name == "c2":
        assert engine.last_path()[0] == 1


@pytest.mark.parametrize("name,scale", [("c1", 0.01), ("c2", 0.002), ("c5", 0.002)])
@pytest.mark.parametrize("range_bytes", [16, 64, 128])
def test_tiny_ranges_fall_back_or_match(engine, name, scale, range_bytes):
    """Ranges shorter than a record: wrong speculation is caught by the chain check (auto path)."""
    from paper_2504_03683_b200 import synth

    _run(engine, synth.config(name, scale), range_bytes)


@pytest.mark.parametrize("range_bytes", [0, 512, 2048])
@pytest.mark.parametrize("seed", range(6))
def test_single_pass_adversarial(engine, seed, range_bytes):
    """Orphans, typed mismatches, unclosed calls, equal timestamps, deep stacks (overflow chunks)."""
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    params = dict(orphan_p=0.01 * seed, mismatch_p=0.02 * (seed % 3), meta_p=0.03, close_at_end=seed % 2,
                  max_depth=[4, 8, 64, 300, 2, 16][seed], push_p=[0.5, 0.6, 0.7, 0.9, 0.5, 0.55][seed],
                  gap_lo=0, gap_hi=[3, 600, 1, 50, 0, 5][seed], prof_p=0.3)
    streams = [synth.StreamSpec(f"h{i % 3}", P + 100 * (i % 4), P + 100 * (i % 4) + i, 3000 + 997 * i,
                                9000 + 31 * seed + i) for i in range(12)]
    wl = synth.Workload(f"adv{seed}", synth.ze_registry(), streams, params, kernel_names=synth.kernel_pool(30))
    _run(engine, wl, range_bytes)


def test_single_pass_is_taken_on_clean_traces(engine):
    from paper_2504_03683_b200 import synth

    before = engine.last_path()[1]
    _run(engine, synth.config("c2", 0.002))
    path, fallbacks, rb = engine.last_path()
    assert path == 1 and fallbacks == before and rb >= 1024


def test_error_traces_fall_back_to_exact_path(engine):
    """A corrupt record: the single pass flags it, the exact path names the error."""
    from paper_2504_03683_b200 import synth

    wl = synth.config("c2", 0.001)
    raws = synth.generate(wl)
    bad = bytearray(raws[7].data)
    bad[16 + 40 * 16] ^= 0xFF  # scramble a byte somewhere inside the stream
    from paper_2504_03683_b200.tracefile import RawStream

    r = raws[7]
    raws[7] = RawStream(r.hostname, r.pid, r.tid, r.name, bytes(bad), r.info)
    from oracle import oracle

    infos = [x.info for x in raws]
    got = engine.run(raws, wl.registry, infos)
    want = oracle.run(raws, wl.registry, infos)
    assert (got.error is None) == (want.error is None)
    if want.error is not None:
        assert type(got.error) is type(want.error) and str(got.error) == str(want.error)
        assert engine.last_path()[0] == 0
    else:
        assert got.report == want.report and got.stats == want.stats


@pytest.mark.parametrize("max_depth,push_p", [(64, 0.55), (300, 0.9)])
def test_deep_stacks_second_run_inline(engine, max_depth, push_p):
    """The first run of a deep trace spills stacks to overflow chunks through the slow path; the
    context then switches to the kernel variant that keeps them inline: both runs match the oracle."""
    from oracle import oracle
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    streams = [synth.StreamSpec("h", P, P + i, 20000 + 3001 * i, 7100 + i) for i in range(6)]
    wl = synth.Workload("deep", synth.ze_registry(), streams,
                        dict(max_depth=max_depth, push_p=push_p, mismatch_p=0.01, close_at_end=0, prof_p=0.2),
                        kernel_names=synth.kernel_pool(12))
    raws = synth.generate(wl)
    infos = [r.info for r in raws]
    want = oracle.run(raws, wl.registry, infos)
    for i in range(2):
        got = engine.run(raws, wl.registry, infos, reuse_streams=i > 0)
        assert engine.last_path()[0] == 1
        assert got.stats == want.stats and got.report == want.report and got.orphans == want.orphans


@pytest.mark.parametrize("name,scale,prof_p", [("c5", 0.004, None), ("c2", 0.003, 0.6), ("c4", 0.003, 0.9)])
def test_device_heavy_repeated_runs(engine, name, scale, prof_p):
    """Device-heavy traces run repeatedly on the same staged streams (the CTA name caches and
    the global name dictionary start over each run): every run matches the oracle."""
    import dataclasses

    from oracle import oracle
    from paper_2504_03683_b200 import synth

    wl = synth.config(name, scale)
    if prof_p is not None:
        wl = dataclasses.replace(wl, params=dict(wl.params, prof_p=prof_p))
    raws = synth.generate(wl)
    infos = [r.info for r in raws]
    want = oracle.run(raws, wl.registry, infos)
    for i in range(3):
        got = engine.run(raws, wl.registry, infos, reuse_streams=i > 0)
        assert engine.last_path()[0] == 1
        assert got.stats == want.stats and got.report == want.report and got.orphans == want.orphans


@pytest.mark.parametrize("n_top,n_low", [(1000, 1000), (3000, 1500)])
@pytest.mark.parametrize("range_bytes", [0, 1008])
def test_large_registry_deep_stacks(engine, n_top, n_low, range_bytes):
    """Large registries (max schema id >= 512): descriptors as 4-byte compact entries in shared
    memory (functions >= 0xFFF and the variable-field annotation schema keep the uint4 read through
    L1); depth-64 stacks in the shared top window with older entries spilled.  Three runs on the same
    streams (the first picks the overflow-chunk kernel variant for the next) match the oracle."""
    from oracle import oracle
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.engine import OPT_PATH, OPT_RANGE_BYTES

    reg = synth.layered_registry(n_top=n_top, n_low=n_low)
    layers = {s.function: (0 if s.function.startswith("sycl") else 1)
              for s in reg.schemas if s.event_class == "host_entry"}
    P = synth.PID_BASE
    streams = [synth.StreamSpec("h", P, P + i, 6000 + 1501 * i, 9100 + i) for i in range(8)]
    wl = synth.Workload("big", reg, streams, {"max_depth": 64, "push_p": 0.55, "zipf_s": 1.1, "n_layers": 2,
                                              "mismatch_p": 0.002, "close_at_end": 0}, layers=layers)
    raws = synth.generate(wl)
    infos = [r.info for r in raws]
    want = oracle.run(raws, wl.registry, infos)
    engine.set_option(OPT_PATH, 2)
    engine.set_option(OPT_RANGE_BYTES, range_bytes)
    try:
        for i in range(3):
            got = engine.run(raws, wl.registry, infos, reuse_streams=i > 0)
            assert engine.last_path()[0] == 1
            assert got.stats == want.stats and got.report == want.report and got.orphans == want.orphans
    finally:
        engine.set_option(OPT_PATH, 0)
        engine.set_option(OPT_RANGE_BYTES, 0)


def _shift_ids(wl, raws, delta):
    """The same workload with every schema id moved up by `delta` (registry and record headers)."""
    import dataclasses
    import struct

    from paper_2504_03683_b200.registry import SchemaRegistry

    doc = wl.registry.to_dict()
    for s in doc["schemas"]:
        s["id"] += delta
    reg = SchemaRegistry.from_dict(doc)
    out = []
    for r in raws:
        d = bytearray(r.data)
        o = 16
        while o + 16 <= len(d):
            sid, _ts, plen = struct.unpack_from("<IQI", d, o)
            struct.pack_into("<I", d, o, sid + delta)
            o += 16 + plen
        out.append(dataclasses.replace(r, data=bytes(d)) if dataclasses.is_dataclass(r) else r._replace(data=bytes(d)))
    return dataclasses.replace(wl, registry=reg), out


@pytest.mark.parametrize("name,scale", [("c5", 0.002), ("c2", 0.002)])
def test_sparse_ids_device_registry(engine, name, scale):
    """Schema ids above kSdescMax with device-profiling schemas: compact descriptors for the fixed
    host records, the uint4 through L1 for variable ones (device records, strings), the CTA name
    cache kept; tally, stats and orphans match the oracle on both runs of the same streams."""
    from oracle import oracle
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.engine import OPT_PATH

    wl = synth.config(name, scale)
    wl, raws = _shift_ids(wl, synth.generate(wl), 1000)
    infos = [r.info for r in raws]
    want = oracle.run(raws, wl.registry, infos)
    engine.set_option(OPT_PATH, 2)
    try:
        for i in range(2):
            got = engine.run(raws, wl.registry, infos, reuse_streams=i > 0)
            assert engine.last_path()[0] == 1
            assert got.stats == want.stats and got.report == want.report and got.orphans == want.orphans
    finally:
        engine.set_option(OPT_PATH, 0)

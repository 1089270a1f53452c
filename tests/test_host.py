"""CPU tests of the product's host side: the instance generator, degrade,
validation and the reference layout (csrc/host_gen.cpp), each bit-exact
against the reference (oracle/_ref) or the committed golden fixtures, and
the multi-GPU shard partition."""
import os
import struct

import numpy as np
import pytest

import paper_2509_10722_b200 as pmp
from paper_2509_10722_b200.shard import local_shard, shard_bounds

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _spec(m, n, avg, kind, weights, seed):
    w = pmp.WeightDist.constant(weights[1]) if weights[0] == "constant" else pmp.WeightDist.uniform(weights[1], weights[2])
    return pmp.GenSpec(m=m, n=n, avg_links_per_stream=avg, kind=pmp.GenKind(kind), weights=w, seed=seed)


GEN_CASES = [
    (1000, 10000, 5.0, 0, ("constant", 1.0, 1.0), 7),   # config A
    (300, 150, 4.0, 2, ("uniform", 0.5, 1.5), 3),
    (40, 20, 4.0, 2, ("constant", 1.0, 1.0), 9),
    (200, 0, 10.0, 1, ("uniform", 0.0, 2.0), 5),          # n = 0 -> m/2, linear
    (50, 30, 80.0, 0, ("constant", 2.0, 2.0), 1),         # routes capped at m
]


@pytest.mark.parametrize("case", GEN_CASES)
def test_generator_bit_exact_with_reference(case, reference):
    ra = reference.gen(*case).arrays()
    p = pmp.gen_uncongested(_spec(*case))
    assert (p.m, p.n, p.nnz) == (ra.m, ra.n, ra.nnz)
    for mine, theirs in [(p.stream_offsets, ra.stream_offsets), (p.route_links, ra.route_links),
                         (p.weights, ra.weights), (p.kinds, ra.kinds), (p.capacities, ra.capacities)]:
        np.testing.assert_array_equal(mine, theirs)


def test_config_b_nnz_matches_survey():
    # config B has nnz 10,002,286
    p = pmp.gen_uncongested(_spec(100000, 1000000, 10.0, 0, ("constant", 1.0, 1.0), 7))
    assert p.nnz == 10002286


@pytest.mark.parametrize("case,hot,threads", [
    ((2000, 30000, 5.0, 2, ("uniform", 0.5, 1.5), 21), (0.01, 0.1), "7"),
    ((2000, 30000, 5.0, 0, ("constant", 1.0, 1.0), 4), (0.02, 0.3), "1"),
    ((300, 1000, 20.0, 1, ("constant", 1.0, 1.0), 8), (0.5, 0.9), "16"),   # hot links already on routes
    ((50, 7, 3.0, 2, ("constant", 1.0, 1.0), 2), (1.0, 1.0), "3"),          # every link hot, every draw hits
])
def test_congested_generator_parallel_draws_bit_exact(case, hot, threads, reference, monkeypatch):
    # the hot phase draws from jumped mt19937_64 engines on several threads
    # (csrc/host_mt.h); ranges split hot links' runs at arbitrary streams
    monkeypatch.setenv("NUMPMP_HOST_THREADS", threads)
    ra = reference.gen(*case, congested=True, hot_link_fraction=hot[0], hot_stream_fraction=hot[1]).arrays()
    p = pmp.gen_congested(_spec(*case), *hot)
    assert p.nnz == ra.nnz
    np.testing.assert_array_equal(p.stream_offsets, ra.stream_offsets)
    np.testing.assert_array_equal(p.route_links, ra.route_links)
    np.testing.assert_array_equal(p.weights, ra.weights)
    np.testing.assert_array_equal(p.capacities, ra.capacities)


@pytest.mark.slow
def test_congested_generator_config_f_bit_exact(reference):
    # bench config F (1e8 hot-phase draws, 2e7 nonzeros): the jumped, threaded draws at scale
    case = (100000, 1000000, 10.0, 2, ("uniform", 0.5, 1.5), 7)
    ra = reference.gen(*case, congested=True, hot_link_fraction=0.001, hot_stream_fraction=0.1).arrays()
    p = pmp.gen_congested(_spec(*case), 0.001, 0.1)
    assert p.nnz == ra.nnz
    np.testing.assert_array_equal(p.stream_offsets, ra.stream_offsets)
    np.testing.assert_array_equal(p.route_links, ra.route_links)


def test_congested_generator_bit_exact(reference):
    case = (400, 300, 4.0, 2, ("uniform", 0.5, 1.5), 13)
    ra = reference.gen(*case, congested=True, hot_link_fraction=0.01, hot_stream_fraction=0.2).arrays()
    p = pmp.gen_congested(_spec(*case), 0.01, 0.2)
    np.testing.assert_array_equal(p.stream_offsets, ra.stream_offsets)
    np.testing.assert_array_equal(p.route_links, ra.route_links)
    np.testing.assert_array_equal(p.capacities, ra.capacities)


@pytest.mark.parametrize("args", [
    (12, 24, 5.0, 30, 40, 3, 24, 50.0, 4),
    (100, 192, 5.0, 952, 110, 3, 60, 50.0, 4),       # the paper's transit case
    (30, 48, 5.0, 80, 300, 5, 48, 20.0, 9),
])
def test_transit_generator_bit_exact(args, reference):
    p, dropped = pmp.gen_transit(pmp.TransitSpec(*args))
    rp = reference.gen_transit(*args)
    ra = rp.arrays()
    assert dropped == rp.dropped
    for mine, theirs in [(p.stream_offsets, ra.stream_offsets), (p.route_links, ra.route_links),
                         (p.capacities, ra.capacities), (p.weights, ra.weights), (p.kinds, ra.kinds)]:
        np.testing.assert_array_equal(mine, theirs)


@pytest.mark.slow
def test_transit_config_e_bit_exact(reference):
    # BASELINE.json configs[4]: m 182,784, n 16,923,949, nnz 51,702,844
    args = (100, 192, 5.0, 952, 9900, 9, 192, 50.0, 4)
    p, dropped = pmp.gen_transit(pmp.TransitSpec(*args))
    assert (p.m, p.n, p.nnz, dropped) == (182784, 16923949, 51702844, 183251)
    ra = reference.gen_transit(*args).arrays()
    np.testing.assert_array_equal(p.route_links, ra.route_links)
    np.testing.assert_array_equal(p.stream_offsets, ra.stream_offsets)


def test_degrade_bit_exact(reference):
    case = (500, 2000, 6.0, 2, ("uniform", 0.5, 1.5), 17)
    rd = reference.gen(*case).degrade(0.5, 0.5, 99).arrays()
    p = pmp.degrade(pmp.gen_uncongested(_spec(*case)), 0.5, 0.5, 99)
    np.testing.assert_array_equal(p.capacities, rd.capacities)


@pytest.mark.parametrize("p_fail,seed", [(0.25, 0), (0.1, 9)])
def test_fail_and_prune_bit_exact(reference, p_fail, seed):
    # gen.hpp:181-223 and the PruneMap of gen.hpp:146-178
    case = (400, 1500, 4.0, 2, ("uniform", 0.5, 1.5), 5)
    rp = reference.gen(*case).fail_and_prune(p_fail, seed)
    ra = rp.arrays()
    lm, sm = rp.prune_maps()
    q, mp = pmp.fail_and_prune(pmp.gen_uncongested(_spec(*case)), p_fail, seed)
    assert (q.m, q.n, q.nnz) == (rp.m, rp.n, rp.nnz)
    for mine, theirs in [(q.stream_offsets, ra.stream_offsets), (q.route_links, ra.route_links),
                         (q.capacities, ra.capacities), (q.weights, ra.weights), (q.kinds, ra.kinds),
                         (mp.link_map, lm), (mp.stream_map, sm)]:
        np.testing.assert_array_equal(mine, theirs)


@pytest.mark.parametrize("name", ["config_a", "mixed_small", "transit_small"])
def test_host_layout_matches_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    nnz = int(z["stream_offsets"][-1])
    p = pmp.Problem(int(z["m"]), int(z["n"]), z["capacities"], z["weights"], z["kinds"], z["stream_offsets"],
                    z["terminal_link"][:nnz])
    L = p.layout
    np.testing.assert_array_equal(L.terminal_link, z["terminal_link"])
    np.testing.assert_array_equal(L.link_offsets, z["link_offsets"])
    np.testing.assert_array_equal(L.link_terminals, z["link_terminals"])
    np.testing.assert_array_equal(L.link_counts, z["link_counts"])
    assert L.slack_terminal(3) == nnz + 3


def test_bipartite_fixture_counts():
    # test_model.cpp:19-31
    S = pmp.Stream
    p = pmp.build_problem([S(0, pmp.StreamKind.Log, "", 1.0, [0]), S(1, pmp.StreamKind.Log, "", 1.0, [1, 2]),
                           S(2, pmp.StreamKind.Log, "", 1.0, [1])], [1.0, 1.0, 1.0])
    assert (p.m, p.n, p.nnz, p.total_terminals) == (3, 3, 4, 7)
    assert list(p.layout.link_counts) == [2, 3, 2]


INVALID = [
    # (routes, kinds, weights, caps) -- model.hpp:76-155 rules
    ([[0, 0]], [0], [1.0], [1.0]),                 # distinct-links
    ([[]], [0], [1.0], [1.0]),                     # non-empty-route
    ([[3]], [0], [1.0], [1.0]),                    # link-in-range
    ([[0]], [0], [1.0], [0.0, 1.0, 1.0]),          # positive-capacity
    ([[0]], [0], [0.0], [1.0]),                    # positive-log-weight
    ([[0]], [1], [-1.0], [1.0]),                   # nonnegative-weight
    ([[0]], [0], [float("nan")], [1.0]),           # finite-weight
    ([[0]], [0], [1.0], [float("inf")]),           # positive-capacity (non-finite)
    ([[0, 0], [5], [1, 1]] * 4, [0] * 12, [1.0] * 12, [1.0, -1.0]),  # > 8 violations
]


@pytest.mark.parametrize("case", INVALID)
def test_validation_messages_match_reference(case, reference):
    routes, kinds, weights, caps = case
    offs = np.cumsum([0] + [len(r) for r in routes]).astype(np.int64)
    rl = np.array([x for r in routes for x in r], np.int32)
    out = reference.build_problem(len(caps), len(routes), offs, rl, kinds, weights, caps)
    assert isinstance(out, tuple) and out[0] == 2, out  # ValidationError
    with pytest.raises(pmp.ValidationError) as ei:
        pmp.problem_from_arrays(len(caps), len(routes), caps, weights, kinds, offs, rl)
    assert str(ei.value) == out[1]


def test_build_problem_rejects_empty():
    with pytest.raises(pmp.ValidationError):
        pmp.build_problem([], [1.0])
    with pytest.raises(pmp.ValidationError):
        pmp.build_problem([pmp.Stream(0, pmp.StreamKind.Log, "", 1.0, [0])], [])


def test_generator_spec_errors():
    with pytest.raises(pmp.GenError):
        pmp.gen_uncongested(pmp.GenSpec(m=0))
    with pytest.raises(pmp.GenError):
        pmp.gen_uncongested(pmp.GenSpec(m=10, avg_links_per_stream=0.5))
    with pytest.raises(pmp.GenError):
        pmp.gen_uncongested(pmp.GenSpec(m=10, weights=pmp.WeightDist.uniform(2.0, 1.0)))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_bounds_tile_and_balance(world):
    p = pmp.gen_uncongested(_spec(1000, 10000, 5.0, 2, ("uniform", 0.5, 1.5), 7))
    b = shard_bounds(p.stream_offsets, world)
    assert b[0] == 0 and b[-1] == p.n and np.all(np.diff(b) >= 0)
    loads = np.diff(p.stream_offsets[b])
    assert loads.sum() == p.nnz
    assert loads.max() - loads.min() <= 2 * int(np.max(np.diff(p.stream_offsets)))  # within one stream's route
    parts = [local_shard(p, r, world) for r in range(world)]
    np.testing.assert_array_equal(np.concatenate([q.route_links for q, _ in parts]), p.route_links)
    np.testing.assert_array_equal(np.concatenate([q.weights for q, _ in parts]), p.weights)
    assert [s0 for _, s0 in parts] == list(b[:-1])
    for q, _ in parts:
        assert q.stream_offsets[0] == 0 and q.m == p.m


# ------------------------------------------------------ problem files (io.hpp)
@pytest.mark.parametrize("encoding", ["text", "binary"])
def test_problem_files_match_reference(reference, tmp_path, encoding):
    # io.hpp:126-279: the reference's file read by ours gives its Problem,
    # and ours writes the reference's bytes
    case = (400, 1500, 4.0, 2, ("uniform", 0.5, 1.5), 5)
    rp = reference.gen(*case)
    ra = rp.arrays()
    f_ref = str(tmp_path / ("ref." + encoding))
    rp.write_problem(f_ref, encoding)
    q = pmp.read_problem(f_ref)
    nnz = int(ra.stream_offsets[-1])
    for mine, theirs in [(q.stream_offsets, ra.stream_offsets), (q.route_links, ra.terminal_link[:nnz]),
                         (q.capacities, ra.capacities), (q.weights, ra.weights), (q.kinds, ra.kinds)]:
        np.testing.assert_array_equal(mine, theirs)
    f_ours = str(tmp_path / ("ours." + encoding))
    pmp.write_problem(q, f_ours, encoding)
    assert open(f_ours, "rb").read() == open(f_ref, "rb").read()


BAD_FILES = [
    b"NUMP 2 1 1\n1\nlog 1 1 0\n",
    b"NUMP 1 2 1\n1\nlog 1 1 0\n",
    b"NUMP 1 1 1\n1.5x\nlog 1 1 0\n",
    b"NUMP 1 1 1\n1\nfoo 1 1 0\n",
    b"NUMP 1 1 1\n1\nlog 1 2 0\n",
    b"NUMP 1 1 2\n1\nlog 1 1 0\n",
    b"NUMP 1 1 1\n1\nlog 1 1 0\n\nlog 1 1 0\n",
    b"NUMP 1 1 1\n1\nlog 1\n",
    b"NUMP 1 0 1\n",
    b"NUMP 1 2 1\n1 1\nlog 1 2 0 0\n",       # duplicate link: ValidationError
    b"NUMP 1 1 1\n-1\nlog 1 1 0\n",          # capacity <= 0: ValidationError
    b"NUMPB 1\n\x01\x00\x00\x00\x00\x00\x00\x00",  # truncated header
    b"NUMPB 1\n" + (1).to_bytes(8, "little") + (1).to_bytes(8, "little") + struct.pack("<d", 1.0)
    + b"\x07",  # unknown kind
    b"NUMPB 1\n" + (1).to_bytes(8, "little") + (1).to_bytes(8, "little") + struct.pack("<d", 1.0)
    + b"\x00" + struct.pack("<d", 1.0) + (3).to_bytes(8, "little") + (0).to_bytes(8, "little"),  # truncated route
]


@pytest.mark.parametrize("blob", BAD_FILES)
def test_problem_file_errors_match_reference(reference, tmp_path, blob):
    f = str(tmp_path / "bad.nump")
    open(f, "wb").write(blob)
    with pytest.raises(RuntimeError) as theirs:
        reference.read_problem(f)
    with pytest.raises((pmp.IoError, pmp.ValidationError)) as mine:
        pmp.read_problem(f)
    assert str(theirs.value).split(": ", 1)[1] == str(mine.value)


@pytest.mark.slow
def test_binary_reader_config_c_scale(tmp_path):
    # the reference reads config C in 11.9 s single-threaded
    import time

    p = pmp.gen_uncongested(_spec(1000000, 10000000, 10.0, 2, ("uniform", 0.5, 1.5), 7))
    f = str(tmp_path / "c.numpb")
    pmp.write_problem(p, f, "binary")
    t = time.perf_counter()
    q = pmp.read_problem(f)
    dt = time.perf_counter() - t
    np.testing.assert_array_equal(q.route_links, p.route_links)
    np.testing.assert_array_equal(q.stream_offsets, p.stream_offsets)
    print(f"read_problem config C: {dt:.2f} s")


@pytest.mark.parametrize("m,world", [(1, 1), (10, 3), (1000000, 8), (182784, 8), (7, 8)])
def test_link_owner_ranges_cover_the_links(m, world):
    # the peer-memory exchange's owner partition (csrc/pmp_solver.cu
    # create_impl: mo = ceil(m / world), rank q owns [q*mo, min(m, (q+1)*mo)))
    from paper_2509_10722_b200.shard import link_owners

    b = link_owners(m, world)
    assert b[0] == 0 and b[-1] == m and len(b) == world + 1
    assert np.all(np.diff(b) >= 0)
    mo = -(-m // world)
    for l in (0, m // 2, m - 1):  # owner(l) = l // mo lands in its range
        q = l // mo
        assert b[q] <= l < b[q + 1]


def test_algorithmic_bytes_match_survey():
    # B_alg = 8 nnz + 45 n + 76 m (+8) per iteration
    import bench

    k1, k2 = bench.alg_bytes(1000000, 10000000, 100006749)
    assert k1 + k2 == 8 * 100006749 + 45 * 10000000 + 76 * 1000000 + 8


# ------------------------------------------------- reports
TRANSIT_REPORT_CASES = [
    (12, 24, 5.0, 30, 40, 3, 24, 50.0, 4),
    (30, 48, 5.0, 80, 300, 5, 48, 20.0, 9),
]


@pytest.mark.parametrize("args", TRANSIT_REPORT_CASES)
def test_transit_metadata_bit_exact(args, reference):
    p, meta = pmp.gen_transit(pmp.TransitSpec(*args), with_meta=True)
    od, route, t0, origin, dest = reference.gen_transit(*args).transit_meta()
    np.testing.assert_array_equal(meta.stream_od, od)
    np.testing.assert_array_equal(meta.stream_route, route)
    np.testing.assert_array_equal(meta.stream_t0, t0)
    np.testing.assert_array_equal(meta.od_origin, origin)
    np.testing.assert_array_equal(meta.od_dest, dest)
    assert meta.dropped_streams == pmp.gen_transit(pmp.TransitSpec(*args))[1]


def test_transit_metadata_rejects_other_instances():
    from paper_2509_10722_b200 import _lib

    L = _lib.lib()
    import ctypes as C

    inst = C.c_void_p()
    assert L.numpmp_gen_uncongested(C.byref(_spec(40, 20, 4.0, 2, ("constant", 1.0, 1.0), 9)._c()),
                                    C.byref(inst)) == 0
    k = C.c_int64()
    assert L.numpmp_transit_meta(inst, C.byref(k), None, None, None, None, None) == 2
    assert b"not a transit instance" in L.numpmp_host_last_error()
    L.numpmp_instance_free(inst)


@pytest.mark.parametrize("args", TRANSIT_REPORT_CASES)
def test_transit_report_matches_reference(args, reference, tmp_path):
    p, meta = pmp.gen_transit(pmp.TransitSpec(*args), with_meta=True)
    rp = reference.gen_transit(*args)
    rng = np.random.default_rng(5)
    x = rng.random(p.n) * 3.0
    lam = rng.random(p.m) * 0.2
    lam[rng.random(p.m) < 0.4] = 0.0  # uncongested links price at zero
    checked = 0
    for od in range(len(meta.od_origin)):
        for t0 in sorted(set(meta.stream_t0[meta.stream_od == od].tolist()))[:3]:
            rows = pmp.transit_report(p, x, lam, meta, od, t0)
            theirs = str(tmp_path / "ref.csv")
            stream, pi, hats = rp.transit_report(x, lam, od, t0, theirs)
            assert [r.stream for r in rows] == stream.tolist()
            assert [r.pi for r in rows] == pi.tolist()  # bit-exact route-order sums
            for r, h in zip(rows, hats):
                assert r.lambda_hat == h.tolist()
            mine = str(tmp_path / "mine.csv")
            pmp.write_transit_report_csv(rows, mine)
            assert open(mine, "rb").read() == open(theirs, "rb").read()
            checked += len(rows)
    assert checked > 0
    # a departure bin with no stream: empty report, header only
    assert pmp.transit_report(p, x, lam, meta, 0, -1) == []


def test_transit_report_errors(reference, tmp_path):
    args = TRANSIT_REPORT_CASES[0]
    p, meta = pmp.gen_transit(pmp.TransitSpec(*args), with_meta=True)
    k = len(meta.od_origin)
    x, lam = np.ones(p.n), np.zeros(p.m)
    # std::invalid_argument in the reference (transit.hpp:343,349) -> ValueError
    with pytest.raises(ValueError, match=rf"^unknown OD id {k}; available: 0\.\.{k - 1}$"):
        pmp.transit_report(p, x, lam, meta, k, 0)
    with pytest.raises(RuntimeError, match=rf"unknown OD id {k}; available: 0\.\.{k - 1}$"):
        reference.gen_transit(*args).transit_report(x, lam, k, 0, str(tmp_path / "r.csv"))
    with pytest.raises(ValueError, match="metadata does not match problem"):
        q = pmp.gen_uncongested(_spec(40, 20, 4.0, 2, ("constant", 1.0, 1.0), 9))
        pmp.transit_report(q, np.ones(q.n), np.zeros(q.m), meta, 0, 0)
    # all prices zero: normalized prices are 0 (transit.hpp:318-320)
    rows = pmp.transit_report(p, x, lam, meta, 0, int(meta.stream_t0[meta.stream_od == 0][0]))
    assert rows and all(v == 0.0 for r in rows for v in r.lambda_hat)


def test_trace_csv_bytes_match_reference(reference, tmp_path):
    from oracle.oracle import ref_write_trace_csv

    rng = np.random.default_rng(3)
    k = 40
    it = np.cumsum(rng.integers(1, 20, k))
    r, s = rng.random(k) * 1e-3, rng.random(k) ** 7
    rho = 1000.0 * 2.0 ** rng.integers(-5, 5, k)
    obj = -rng.random(k) * 1e6
    r[3], s[4], obj[5], obj[6] = 0.0, 5e-324, -0.0, 1.0 / 3.0
    trace = [pmp.TraceRecord(int(it[i]), r[i], s[i], rho[i], obj[i]) for i in range(k)]
    mine, theirs = str(tmp_path / "mine.csv"), str(tmp_path / "ref.csv")
    pmp.write_trace_csv(trace, mine)
    ref_write_trace_csv(reference, theirs, it, r, s, rho, obj)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    pmp.write_trace_csv([], mine)
    assert open(mine, "rb").read() == b"iter,r_norm,s_norm,rho,objective\n"
    with pytest.raises(pmp.IoError, match=r"^cannot write '/nonexistent/dir/t\.csv'$"):
        pmp.write_trace_csv(trace, "/nonexistent/dir/t.csv")


@pytest.mark.parametrize("args", TRANSIT_REPORT_CASES)
def test_transit_metadata_file_matches_reference(args, reference, tmp_path):
    # io.hpp:444-540: the NUMT sidecar, byte-identical, and read back
    p, meta = pmp.gen_transit(pmp.TransitSpec(*args), with_meta=True)
    mine, theirs = str(tmp_path / "mine.numt"), str(tmp_path / "ref.numt")
    pmp.write_transit_metadata(meta, mine)
    reference.gen_transit(*args).write_transit_metadata(theirs)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    back = pmp.read_transit_metadata(mine)
    for f in ("stream_od", "stream_route", "stream_t0", "od_origin", "od_dest", "edges", "od_route_ptr", "route_ptr",
              "route_edges"):
        np.testing.assert_array_equal(getattr(back, f), getattr(meta, f))
    assert (back.stations, back.time_bins, back.bin_minutes, back.seats, back.dropped_streams) == \
        (meta.stations, meta.time_bins, meta.bin_minutes, meta.seats, meta.dropped_streams)
    # the report from the read-back metadata is the same
    x, lam = np.linspace(0.5, 2.0, p.n), np.linspace(0.0, 1.0, p.m)
    t0 = int(meta.stream_t0[0])
    assert pmp.transit_report(p, x, lam, back, 0, t0) == pmp.transit_report(p, x, lam, meta, 0, t0)


def test_transit_metadata_reader_errors_match_reference(reference, tmp_path):
    from oracle.oracle import Reference  # noqa: F401 (reference fixture already built)

    good = str(tmp_path / "good.numt")
    p, meta = pmp.gen_transit(pmp.TransitSpec(*TRANSIT_REPORT_CASES[0]), with_meta=True)
    pmp.write_transit_metadata(meta, good)
    lines = open(good).read().split("\n")
    n_edges = int(lines[0].split()[4])
    cases = {
        "magic": ["NUMX" + lines[0][4:]] + lines[1:],
        "version": [lines[0].replace("NUMT 1", "NUMT 2", 1)] + lines[1:],
        "head_int": [lines[0].replace("NUMT 1 ", "NUMT 1 x", 1)] + lines[1:],
        "extra": [lines[0], "5 50"] + lines[2:],
        "extra_num": [lines[0], "5 fifty 0"] + lines[2:],
        "edge": lines[:2] + ["1 2 3"] + lines[3:],
        "od": lines[:2 + n_edges] + ["1 2"] + lines[3 + n_edges:],
        "route_len": lines[:3 + n_edges] + ["9 1 2"] + lines[4 + n_edges:],
        "stream": lines[:-3] + ["1 2"] + lines[-2:],
        "truncated": lines[: len(lines) // 2],
    }
    for name, ls in cases.items():
        path = str(tmp_path / f"{name}.numt")
        with open(path, "w") as f:
            f.write("\n".join(ls))
        rc = reference.L.ref_check_transit_metadata(os.fsencode(path))
        assert rc != 0, name
        want = reference.L.ref_last_error().decode()
        with pytest.raises(pmp.IoError) as e:
            pmp.read_transit_metadata(path)
        assert str(e.value) == want, name
    with pytest.raises(pmp.IoError, match=r"^cannot open '/nonexistent/m\.numt'$"):
        pmp.read_transit_metadata("/nonexistent/m.numt")


def test_bench_reference_arm_is_the_reference_alone():
    # bench.py --impl reference: the reference's own generator and stock
    # PmpSolver::solve() (oracle/_ref); no library of this repo is mapped, and
    # the config object is the one the GPU arm prints.
    import json
    import subprocess
    import sys

    import bench

    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libnumpmp_ref.so")
    if not os.path.exists(ref_so):
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "A",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, check=True)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["repo_libs_loaded"] == ["oracle/_ref/libnumpmp_ref.so"]
    assert line["config"] == bench.bench_config("A", 1000, 10000, 49795)
    assert line["iterations_per_step"] == [423]  # config A converges inside the sample
    assert line["cpu_baseline"]["kind"] == "reference"


def test_group_streams_matches_reference(reference):
    # model.hpp:255-286: (tau, kind) partition, ordered by tau, kind, first member
    for args in [(100, 50, 5.0, 2, ("uniform", 0.5, 1.5), 1), (300, 900, 4.0, 2, ("uniform", 0.5, 1.5), 31),
                 (1000, 10000, 5.0, 0, ("constant", 1.0, 1.0), 7)]:
        rp = reference.gen(*args)
        a = rp.arrays()
        p = pmp.problem_from_arrays(a.m, a.n, a.capacities, a.weights, a.kinds, a.stream_offsets, a.route_links)
        got = pmp.group_streams(p)
        want = rp.groups()
        assert len(got) == len(want)
        for g, (tau, kind, members) in zip(got, want):
            assert (g.tau, int(g.kind)) == (tau, kind)
            np.testing.assert_array_equal(g.members, members)
            np.testing.assert_array_equal(g.weights, a.weights[members])
            for i in range(g.tau):
                np.testing.assert_array_equal(g.terminal_links[i], a.route_links[a.stream_offsets[members] + i])

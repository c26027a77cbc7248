"""Known-answer tests from the reference's SPEC (SPEC.md:111-131
configurator, :180-209 MIG slot model, :254-283 allocator), encoded against
this package's public API (the drop-in boundary).  Expected values were
checked against the reference itself (`migplan`); where the SPEC's prose
and the reference code disagree, the reference's behaviour is asserted and
the deviation is noted:
  * size-2 segments start at slots {0, 2, 4} in the code (SPEC prose also
    lists 5; SURVEY §8c "size-2@5 correction");
  * the SPEC's optimization example ("two size-1 segments fill the holes")
    meets propose_small_segments' lexicographic minimum (GPCs, count, -k2)
    (allocator.py:319-359), which prefers ONE size-2 segment when its
    throughput covers the freed rate: it moves as a size-2 where a 2-slot
    hole exists, and is skipped with a diagnostic where only two size-1
    holes exist.
The MIG-geometry cases are host code (CPU); the configurator and allocator
cases run the sm_100a kernels (GPU)."""

import dataclasses

import pytest

import paper_2409_14447_b200 as P
from paper_2409_14447_b200 import mig

T = P.Triplet


# ------------------------------------------------------------ MIG (CPU)
def test_spec_mig_start_slots():
    """preference-ordered starts and footprints."""
    assert [o.start for o in mig.allowed_start_slots(7)] == [0]
    assert [o.occupied for o in mig.allowed_start_slots(4)] == [(0, 1, 2, 3)]      # "only slot 0"
    three = mig.allowed_start_slots(3)
    assert [o.start for o in three] == [4, 0] and three[1].blocked == (3,)       # 3@0 blocks slot 3
    assert [o.start for o in mig.allowed_start_slots(2)] == [0, 2, 4]            # (code; SPEC prose adds 5)
    assert [o.start for o in mig.allowed_start_slots(1)] == list(range(7))
    with pytest.raises(P.InvalidSizeError):                                      # "5 or 6 GPCs are not possible"
        mig.allowed_start_slots(5)


def test_spec_mig_place_remove():
    """try_place / remove."""
    g = mig.GpuState(id=0)
    assert g.place("a", 4, 1, 1, 1.0).start_slot == 0                          # empty GPU, size 4 -> slot 0
    assert g.place("b", 3, 1, 1, 1.0).start_slot == 4 and g.num_gpcs == 7       # "4-3" full
    assert g.place("c", 1, 1, 1, 1.0) is None                                   # full: rejection, unchanged
    assert g.num_gpcs == 7
    h = mig.GpuState(id=1)
    h.placements.append(P.Placement("x", 3, 1, 1, 1.0, 0))                       # size 3 at slot 0 (slot 3 BLOCKED)
    assert h.place("y", 1, 1, 1, 1.0).start_slot == 4
    e = mig.GpuState(id=2)
    p = e.place("z", 2, 1, 1, 1.0)
    e.remove(p)
    assert e.slot_map() == [None] * 7                                            # inverse of place
    with pytest.raises(P.PlacementNotFoundError):                               # second remove: not found
        e.remove(p)
    f = mig.GpuState(id=3)
    q = P.Placement("w", 3, 1, 1, 1.0, 0)
    f.placements.append(q)
    f.remove(q)
    assert f.free_slots() == list(range(7))                                     # 0-2 and BLOCKED 3 freed


def test_spec_mig_full_configs():
    """SPEC.md:210-218 / §II-B: exactly 19 full configurations."""
    full = P.enumerate_full_configs()
    sizes = {tuple(sorted((s for _, s in c), reverse=True)) for c in full}   # (start, size) pairs
    assert len(full) == 19
    assert (1, 1, 1, 1, 1, 1, 1) in sizes and (4, 2, 1) in sizes and (4, 1, 1, 1) in sizes


# ------------------------------------------------ configurator (GPU)
def _svc(name, rate, trips, slo=400.0):
    return dataclasses.replace(P.make_service(name, "m", rate, slo), best_triplets=tuple(trips))


@pytest.mark.gpu
def test_spec_triplet_decision():
    """SPEC.md:111-117 (PAPER §III-B InceptionV3 points)."""
    pts = (P.ProfilePoint("m", 1, 4, 1, 354.0, 11.0), P.ProfilePoint("m", 1, 4, 2, 444.0, 18.0),
           P.ProfilePoint("m", 1, 4, 3, 446.0, 27.0))
    tab = P.ProfileTable("m", pts)
    got = P.decide_best_triplets(P.make_service("s", "m", 100.0, 40.0), tab)        # internal latency 20 ms
    assert got.best_triplets == (T(1, 4, 2, 444.0, 18.0),)                          # lat 27 exceeds the bound
    with pytest.raises(P.InfeasibleSLOError):                                       # below every latency
        P.decide_best_triplets(P.make_service("s", "m", 100.0, 20.0), tab)
    single = P.ProfileTable("m", (P.ProfilePoint("m", 1, 1, 1, 10.0, 5.0), P.ProfilePoint("m", 4, 2, 1, 50.0, 6.0)))
    got = P.decide_best_triplets(P.make_service("s", "m", 100.0, 40.0), single)
    assert got.best_triplets == (T(1, 1, 1, 10.0, 5.0), T(4, 2, 1, 50.0, 6.0))    # one qualifying point per size


@pytest.mark.gpu
def test_spec_select_optimal_segment():
    """SPEC.md:118-125."""
    t1, t4 = T(1, 4, 3, 446.0, 27.0), T(4, 8, 3, 1810.0, 13.0)
    assert P.select_optimal_segment([t1, t4]) == t4                                 # 452.5 > 446
    assert P.select_optimal_segment([t1]) == t1                                     # singleton
    a, b = T(1, 1, 1, 100.0, 1.0), T(2, 1, 1, 200.0, 1.0)
    assert P.select_optimal_segment([a, b]) == b                                    # equal ratio: larger size


@pytest.mark.gpu
def test_spec_demand_matching():
    """SPEC.md:126-131 (req_rate 4196 = ResNet-50 in S6, PAPER Table IV)."""
    t1, t4 = T(1, 4, 3, 446.0, 27.0), T(4, 8, 3, 1810.0, 13.0)
    r = P.match_demand(_svc("r", 4196.0, (t1, t4)))
    assert (r.optimal_segment, r.optimal_segment_count, r.last_segment) == (t4, 2, t4)   # 576 > 446
    assert len(r.segments()) == 3 and r.total_gpcs == 12
    r = P.match_demand(_svc("r", 400.0, (t1, t4)))
    assert (r.optimal_segment, r.optimal_segment_count, r.last_segment) == (t4, 0, t1)   # 446 >= 400
    r = P.match_demand(_svc("r", 0.0, (t1, t4)))
    assert r.optimal_segment_count == 0 and r.last_segment is None and r.segments() == ()


# --------------------------------------------------- allocator (GPU)
def _conf(name, opt, count, last=None, extra=()):
    trips = {t.instance_size: t for t in (opt, last, *extra) if t is not None}
    return dataclasses.replace(P.make_service(name, "m", 1.0, 100.0),
                               best_triplets=tuple(trips[s] for s in sorted(trips)), optimal_segment=opt,
                               optimal_segment_count=count, last_segment=last)


def _layout(dmap):
    return [[(p.service_id, p.instance_size, p.start_slot) for p in g.placements] for g in dmap.gpus]


def _t(size, tp=None):
    return T(size, 1, 1, 100.0 * size if tp is None else tp, 1.0)


@pytest.mark.gpu
def test_spec_segment_relocation():
    """first-fit-decreasing with the slot rules."""
    d = P.relocate_segments([_conf("A", _t(4), 1), _conf("B", _t(4), 1), _conf("C", _t(3), 2)])
    assert _layout(d) == [[("A", 4, 0), ("C", 3, 4)], [("B", 4, 0), ("C", 3, 4)]]
    assert d.gpu_count == 2 and d.total_gpcs == 14                                  # 0 free GPCs
    d = P.relocate_segments([_conf("A", _t(7), 1)])
    assert _layout(d) == [[("A", 7, 0)]]
    d = P.relocate_segments([_conf("A", _t(4), 2), _conf("C", _t(3), 2), _conf("D", _t(1), 1)])
    assert _layout(d) == [[("A", 4, 0), ("C", 3, 4)], [("A", 4, 0), ("C", 3, 4)], [("D", 1, 0)]]


@pytest.mark.gpu
def test_spec_allocation_optimization():
    """SPEC.md:261-272.  The last GPU holds B's size-2 segment (tp 200); B's
    size-1 triplet has tp 120.  With a 2-slot hole on GPU 0 (slots 4-5) the
    proposal -- one size-2, (2 GPCs, 1 segment) beats two size-1s (2 GPCs,
    2 segments) -- moves there and the last GPU is removed; with only two
    size-1 holes (slots 5, 6) the size-2 cannot start at 5 and the GPU is
    kept with a diagnostic (the reference's behaviour; see module doc)."""
    t1, t2 = _t(1, 120.0), _t(2, 200.0)
    X, Y, B = _conf("X", _t(4, 400.0), 1), _conf("Y", _t(1, 90.0), 1), _conf("B", t2, 1, extra=(t1,))
    for y_slot, layout, ids, freed, n_diag in ((6, [[("X", 4, 0), ("Y", 1, 6), ("B", 2, 4)]], [0], {"B": 0.0}, 0),
                                               (4, [[("X", 4, 0), ("Y", 1, 4)], [("B", 2, 0)]], [0, 1], {}, 1)):
        g0 = mig.GpuState(id=0, placements=[P.Placement("X", 4, 1, 1, 400.0, 0),
                                            P.Placement("Y", 1, 1, 1, 90.0, y_slot)])
        g1 = mig.GpuState(id=1, placements=[P.Placement("B", 2, 1, 1, 200.0, 0)])
        before = P.DeploymentMap(gpus=[g0, g1])
        out = P.optimize_allocation(before, [X, Y, B], threshold=4)
        assert _layout(out) == layout and [g.id for g in out.gpus] == ids
        assert out.freed_rate == freed and len(out.diagnostics) == n_diag
        assert out.gpu_count <= before.gpu_count
        assert _layout(before)[1] == [("B", 2, 0)]                                  # input not mutated
    full = P.DeploymentMap(gpus=[mig.GpuState(id=0, placements=[P.Placement("A", 7, 1, 1, 700.0, 0)])])
    out = P.optimize_allocation(full, [_conf("A", _t(7, 700.0), 1)], threshold=4)
    assert _layout(out) == [[("A", 7, 0)]]                                          # every GPU full: unchanged
    assert P.optimize_allocation(P.DeploymentMap(), [], threshold=4).gpus == []      # empty map -> empty map


@pytest.mark.gpu
def test_spec_small_segments():
    """SPEC.md:273-279."""
    b = _conf("B", _t(2, 260.0), 1, extra=(_t(1, 120.0),))
    assert P.propose_small_segments(b, 0.0) == []
    assert P.propose_small_segments(b, 200.0) == [_t(2, 260.0)]                    # one size-2 beats two size-1s
    c = _conf("C", _t(1, 120.0), 1)
    assert P.propose_small_segments(c, 100.0) == [_t(1, 120.0)]

"""Host-side plan analysis behind the fused launches (csrc/device/engine.cu DevicePlan::
build_index, via mg_plan_fusion_candidates; CPU only): which delay / reverb slots share a
signal spectrum with the previous long-convolution step, and which steps read exactly the
previous step's rows slot by slot (compressor -> noisegate fusion), checked against a direct
restatement over the RenderData step tables, on consoles, unions and random DAGs."""
import numpy as np
import pytest

from oracle import ref as _ref

CONV = (8, 9)


def expected(rd):
    steps = rd.steps
    share = np.zeros(len(steps), dtype=np.int32)
    reads = np.zeros(len(steps), dtype=bool)

    def single(st):
        slots = st.store_end - st.store_begin
        cnt, src = [0] * slots, [-1] * slots
        for g, a in zip(st.gather, st.aggregate):
            cnt[a] += 1
            src[a] = g
        return [s if c == 1 else -1 for s, c in zip(src, cnt)]

    for k in range(1, len(steps)):
        a, b = steps[k - 1], steps[k]
        na, nb = a.store_end - a.store_begin, b.store_end - b.store_begin
        # dense: slot s of b reads exactly row (first + s), from a's rows in order
        dense = (nb > 0 and len(b.gather) == nb and list(b.aggregate) == list(range(nb))
                 and list(b.gather) == list(range(b.gather[0], b.gather[0] + nb)))
        reads[k] = dense and b.gather[0] == a.store_begin and na == nb
        if int(a.type) in CONV and int(b.type) in CONV and not any(a.store_begin <= g < a.store_end for g in b.gather):
            free = {}
            for q, s in enumerate(single(a)):
                if s >= 0:
                    free.setdefault(s, q)
            n = 0
            for s in single(b):
                if s >= 0 and s in free:
                    del free[s]
                    n += 1
            share[k] = n
    return share, reads


def check(mg, t, e):
    rd = mg.compute_render_data(mg.to_flat(mg.Graph.from_arrays(t, e)))
    got_share, got_reads = rd.fusion_candidates()
    want_share, want_reads = expected(rd)
    assert list(got_share) == list(want_share)
    assert list(got_reads) == list(want_reads)
    return rd, got_share, got_reads


@pytest.mark.skipif(not _ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("tracks,prune,seed", [(16, 0.3, 16), (6, 0.0, 1), (32, 0.5, 3)])
def test_console_fusion_candidates(mg, ref, tracks, prune, seed):
    t, e = ref.console(tracks, prune, seed)
    rd, share, reads = check(mg, t, e)
    types = [int(st.type) for st in rd.steps]
    # every track's compressor reads its EQ's rows, the noisegate the compressor's
    assert reads[types.index(5)] and reads[types.index(6)]
    k = next(i for i in range(1, len(types)) if {types[i - 1], types[i]} == {8, 9})
    if prune == 0.0:  # every track sends to both: all of the second step's slots pair up
        assert share[k] == rd.steps[k].store_end - rd.steps[k].store_begin
    else:
        assert 0 < share[k] <= rd.steps[k].store_end - rd.steps[k].store_begin


@pytest.mark.skipif(not _ref.available(), reason="oracle/_ref not built")
def test_union_and_random_dag_fusion_candidates(mg, ref):
    from paper_2408_03204_b200 import sharding
    members = [ref.console(n, 0.3, s) for n, s in ((4, 1), (9, 2), (5, 3))]
    t, e = sharding.union_arrays(members)
    check(mg, t, e)
    for seed in range(40):
        t, e = ref.random_dag(seed, 4, 40)
        check(mg, t, e)

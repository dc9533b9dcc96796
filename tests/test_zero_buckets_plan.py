"""The bucketed stage-2 step's piece layout (mco_zb_plan, SURVEY 8(e) C4 bookkeeping):
ZeroPlan (parallel.cpp:20-34, checked against the compiled reference) applied inside
every bucket; pieces cover the set exactly once; buckets are multiples of 8 N
elements so every piece but the last bucket's starts 32 B aligned; the footprint
accounting sums the same pieces.  Host arithmetic only (no GPU)."""
import ctypes as C

import pytest

import oracle as O
from paper_2312_00407_b200 import zero
from paper_2312_00407_b200._lib import lib
from paper_2312_00407_b200.optim import Kind, _check


def orc_zero_plan(total, N):
    """ZeroPlan::make restated in oracle/mco_oracle.c (pinned to the reference)."""
    parts, offs = (C.c_uint64 * N)(), (C.c_uint64 * (N + 1))()
    assert O.orc.orc_zero_plan(total, N, parts, offs) == 0
    return list(parts), list(offs)


def plan(P, N, B, k, r):
    Br, nb, bo, bl, o, n = C.c_uint64(), C.c_int(), C.c_uint64(), C.c_uint64(), C.c_uint64(), \
        C.c_uint64()
    _check(lib.mco_zb_plan(P, N, B, k, r, C.byref(Br), C.byref(nb), C.byref(bo), C.byref(bl),
                           C.byref(o), C.byref(n)))
    return Br.value, nb.value, bo.value, bl.value, o.value, n.value


@pytest.mark.parametrize("P,N,B", [(10, 4, 0), (100003, 3, 4096), (1 << 20, 8, 1 << 16),
                                   (999, 8, 10), (6738415616, 8, 1 << 28), (13, 1, 5)])
def test_bucket_pieces_are_zeroplan_per_bucket_and_cover_the_set(P, N, B):
    Br, nb, *_ = plan(P, N, B, 0, 0)
    assert Br % (8 * N) == 0 and Br >= min(B or P, P) and nb == -(-P // Br)
    covered = 0
    for k in ([0, 1, nb // 2, nb - 2, nb - 1] if nb > 64 else range(nb)):
        if k < 0:
            continue
        parts, offs = orc_zero_plan(min(P, (k + 1) * Br) - k * Br, N)
        prev_end = None
        for r in range(N):
            _, _, bo, bl, o, n = plan(P, N, B, k, r)
            assert bo == k * Br and bl == min(P, (k + 1) * Br) - k * Br
            assert (o, n) == (offs[r], parts[r])
            if prev_end is not None:
                assert o == prev_end
            prev_end = o + n
            if k < nb - 1:
                assert (bo + o) % 8 == 0 and n % 8 == 0
        assert prev_end == bl
        covered += bl
    if nb <= 64:
        assert covered == P


def test_plan_rejects_bad_arguments():
    with pytest.raises(Exception, match="bucket / rank out of range"):
        plan(100, 2, 16, 99, 0)
    with pytest.raises(Exception, match="non-empty"):
        plan(0, 2, 16, 0, 0)


def test_footprint_matches_the_plan():
    P, N, B = 1000003, 4, 65536
    fp = zero.BucketedZeroOptimizer.footprint(Kind.ADAN, P, N, B, 2, False)
    Br, nb, *_ = plan(P, N, B, 0, 0)
    own0 = sum(plan(P, N, B, k, 0)[5] for k in range(nb))  # rank 0 owns the most
    assert fp["bucket_elems"] == Br and fp["owned"] == own0
    assert fp["state"] == 4 * own0 * 4 and fp["master"] == own0 * 4
    assert fp["replicas"] == 2 * P and fp["staging"] == 2 * Br * 4

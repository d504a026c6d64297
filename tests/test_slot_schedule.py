"""The slot permutation of the register-V Jacobi tier (psd_rv.cuh
next_slot) is a round-robin tournament: over one sweep of KP-1 steps every
index pair meets exactly once in some slot pair (2i, 2i+1), the slot order is
the identity again at every sweep boundary, and with the V row split over Q
lanes (S = KP/Q >= 4 slots each) exactly one element moves to each neighbour
lane per step.  This pins the schedule the kernel's correctness relies on."""
import re

import pytest


def next_slot_from_source():
    src = open("paper_1609_06068_b200/csrc/psd_rv.cuh").read()
    m = re.search(r"return s == 0 \? 0 : \(s & 1\) \? \(s == 1 \? 2 : s - 2\) : \(s == KP - 2 \? KP - 1 : s \+ 2\);", src)
    assert m, "next_slot formula changed; update this test"

    def ns(s, KP):
        return 0 if s == 0 else (2 if s == 1 else s - 2) if s & 1 else (KP - 1 if s == KP - 2 else s + 2)
    return ns


@pytest.mark.parametrize("KP", [4, 8, 16, 32, 64, 96])
def test_round_robin(KP):
    ns = next_slot_from_source()
    slot_of = list(range(KP))
    seen = set()
    for _ in range(KP - 1):
        at = [None] * KP
        for idx, s in enumerate(slot_of):
            at[s] = idx
        for i in range(KP // 2):
            pair = tuple(sorted((at[2 * i], at[2 * i + 1])))
            assert pair not in seen
            seen.add(pair)
        slot_of = [ns(s, KP) for s in slot_of]
    assert len(seen) == KP * (KP - 1) // 2
    assert slot_of == list(range(KP))


@pytest.mark.parametrize("KP,Q", [(8, 1), (8, 2), (16, 2), (16, 4), (32, 2), (32, 8), (64, 4)])
def test_lane_split_moves(KP, Q):
    ns = next_slot_from_source()
    S = KP // Q
    for j in range(KP):
        q, q2 = j // S, ns(j, KP) // S
        if q2 == q + 1:
            assert j == (q + 1) * S - 2 and ns(j, KP) == (q + 1) * S
        elif q2 == q - 1:
            assert j == q * S + 1 and ns(j, KP) == q * S - 1
        else:
            assert q2 == q

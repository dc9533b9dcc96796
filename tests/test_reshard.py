"""Optimizer-state resharding across world sizes (the reference's
extract_state / load_state name+size contract, parallel.cpp:820-862)."""
import torch

from paper_2312_00407_b200 import zero
from paper_2312_00407_b200.optim import ContractError

import pytest


def _states(P, world):
    plan = zero.ZeroPlan.make(P, world)
    full = {n: torch.arange(P, dtype=torch.float32) * (i + 1) for i, n in enumerate(("m", "v"))}
    return [{"steps": 7, "buffers": {n: full[n][slice(*plan.owned_range(r))].clone()
                                     for n in full}} for r in range(world)], full


@pytest.mark.parametrize("P,a,b", [(10, 4, 3), (1000, 8, 2), (7, 3, 8), (10, 1, 4)])
def test_reshard_roundtrip(P, a, b):
    states, full = _states(P, a)
    new = zero.reshard_state(states, P, b)
    plan = zero.ZeroPlan.make(P, b)
    for r, s in enumerate(new):
        lo, hi = plan.owned_range(r)
        assert s["steps"] == 7
        for n in full:
            assert torch.equal(s["buffers"][n], full[n][lo:hi])
    back = zero.reshard_state(new, P, a)
    for x, y in zip(back, states):
        for n in full:
            assert torch.equal(x["buffers"][n], y["buffers"][n])


def test_reshard_rejects_inconsistent_states():
    states, _ = _states(10, 2)
    states[1]["steps"] = 8
    with pytest.raises(ContractError):
        zero.reshard_state(states, 10, 3)
    states, _ = _states(10, 2)
    states[1]["buffers"]["m"] = states[1]["buffers"]["m"][:-1]
    with pytest.raises(ContractError):
        zero.reshard_state(states, 10, 3)

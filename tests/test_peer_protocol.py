"""CPU checks of the PEER exchange (rbg_desc.comm = PEER).

1. A model of the device protocol under adversarial interleavings.  Rank r's stream runs,
   per iteration t = 1, 2, ... (t = the record tag st->k + 1):
     sweep_t : write its candidate column into its own send slot [t & 1], then store its
               record (tag t) into slot (t & 1, r) of EVERY rank's record array;
     wait_t  : block until rank r's array holds tag t in slots (t & 1, p) for all p;
     imgs_t  : read the records, then (later) the winner's column from the owner's slot.
   Every step of every rank is split into its individual stores / loads and the ranks are
   interleaved at random; every load must return iteration t's data.  This is the argument
   for two slots by tag parity: a slot of parity t & 1 is rewritten only at t + 2, and rank p
   gets there only after every rank's record of t + 1, which each rank publishes after its
   own imgs_t (stream order).  With ONE slot the model finds the overwrite race.
2. The host plumbing over gloo (world size 2): every rank's IPC handle blob reaches every
   rank in rank order (dist.all_gather_bytes / connect_peers).
"""
from __future__ import annotations

import random

import pytest

from test_dist_gloo import WORLD, run_world


def _simulate(world: int, iters: int, seed: int, slots: int = 2) -> None:
    rng = random.Random(seed)
    rec = [[[(0, None)] * world for _ in range(slots)] for _ in range(world)]   # rec[r][par][p]
    col = [[None] * slots for _ in range(world)]                              # col[p][par]

    def program(r):
        for t in range(1, iters + 1):
            par = t % slots
            col[r][par] = ("col", r, t)                       # pack into own send slot
            yield
            for q in range(world):                            # P2P record stores, any order
                rec[q][par][r] = (t, ("rec", r, t))
                yield
            while any(rec[r][par][p][0] != t for p in range(world)):   # wait kernel
                yield "blocked"
            seen = []
            for p in range(world):                            # IMGS: decision
                tag, val = rec[r][par][p]
                assert (tag, val) == (t, ("rec", p, t)), (r, t, p, tag, val)
                seen.append(val)
                yield
            owner = (t * 7 + 3) % world                       # any winner
            for _ in range(3):                                # IMGS: column loads, spread out
                assert col[owner][par] == ("col", owner, t), (r, t, owner, col[owner][par])
                yield

    progs = {r: program(r) for r in range(world)}
    blocked = 0
    while progs:
        r = rng.choice(sorted(progs))
        try:
            blocked = blocked + 1 if next(progs[r]) == "blocked" else 0
        except StopIteration:
            del progs[r]
        assert blocked < 200 * world, "deadlock: every rank waits for a record that never comes"


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_peer_protocol_two_slots_never_race(world):
    for seed in range(60):
        _simulate(world, iters=12, seed=seed)


def test_peer_protocol_one_slot_races():
    """The model is sharp enough to see why the second slot exists."""
    with pytest.raises(AssertionError):
        for seed in range(200):
            _simulate(2, iters=12, seed=seed, slots=1)


class _FakeCtx:
    def __init__(self, rank):
        self.rank = rank
        self.got = None

    def peer_export(self):
        return bytes([self.rank]) * 128

    def peer_connect(self, handles):
        self.got = handles


def _connect(rank):
    from paper_1805_06124_b200 import dist as D
    ctx = D.connect_peers(_FakeCtx(rank))
    return ctx.got


def test_connect_peers_over_gloo():
    res = run_world(_connect)
    for got in res:
        assert got == [bytes([p]) * 128 for p in range(WORLD)]


class _FailingCtx(_FakeCtx):
    def peer_export(self):
        from paper_1805_06124_b200 import rbg
        if self.rank == 1:
            raise rbg.RbgError(rbg.ECUDA, "no IPC here")
        return super().peer_export()


def _connect_failing(rank):
    from paper_1805_06124_b200 import dist as D
    from paper_1805_06124_b200 import rbg
    try:
        D.connect_peers(_FailingCtx(rank))
    except rbg.RbgError as e:
        return e.status
    return None


def test_connect_peers_failure_reaches_every_rank():
    """A rank that cannot export its handles still takes part in the all-gather, and every
    rank raises (bench.py then falls back to the NCCL exchange on all ranks)."""
    from paper_1805_06124_b200 import rbg
    assert run_world(_connect_failing) == [rbg.ESTATE, rbg.ESTATE]


def test_enrich_plan_numbers_appended_blocks_in_rank_order():
    from paper_1805_06124_b200 import dist as D
    counts = [3, 0, 5, 1]
    plans = [D.enrich_plan(counts, r, 1000) for r in range(4)]
    assert plans == [(1000, 1009), (1003, 1009), (1003, 1009), (1008, 1009)]
    # concatenating the blocks in rank order gives ids 1000..1008 without gaps
    ids = [i for r in range(4) for i in range(plans[r][0], plans[r][0] + counts[r])]
    assert ids == list(range(1000, 1009))

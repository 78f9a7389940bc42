"""SimWorld's wire ledger and traffic_stats on CPU tensors, mirroring the
reference's own collective tests (tests/test_collectives.py:211-303 of the
reference): the same programs, the same ledger records and byte totals."""
import numpy as np
import pytest
import torch

from paper_2504_14960_b200 import ClusterModel, SimWorld, VarBuffer, traffic_stats
from paper_2504_14960_b200.errors import ProtocolError


def run_world(n, program, workers=None):
    world = SimWorld(n, device="cpu")
    return world, world.run(program, workers=workers)


def rows(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64))


def _mixed_program(payloads, n):
    def program(ctx):
        half = tuple(range(n // 2)) if ctx.rank < n // 2 else tuple(range(n // 2, n))
        out = ctx.all_to_all_v(half, VarBuffer.from_rows(rows(payloads[ctx.rank]), [1] * (n // 2)))
        red = ctx.all_reduce(tuple(range(n)), out.rows().sum(dim=0), "sum")
        buf, _ = ctx.all_gather_v(half, VarBuffer.from_rows(out.rows()))
        return red, buf.rows()

    return program


def test_ledger_records_match_reference_rules():
    rng = np.random.default_rng(5)
    n = 4
    payloads = [rng.standard_normal((2, 3)) for _ in range(n)]
    world, _ = run_world(n, _mixed_program(payloads, n))
    got = [(r.epoch, r.seq, r.group, r.primitive, r.row_width, r.elements_sent) for r in world.ledger]
    # the reference's SimWorld on the same program: a2a sends 1 of 2 rows off-rank,
    # the 4-rank all_reduce of 3 values charges round(3 * 2 * 3 / 4) = 4 per rank,
    # the gather 2 rows * 1 peer * width 3
    assert got == [
        (1, 0, (0, 1), "all_to_all_v", 3, (3, 3)),
        (1, 0, (0, 1, 2, 3), "all_reduce", 1, (4, 4, 4, 4)),
        (1, 0, (2, 3), "all_to_all_v", 3, (3, 3)),
        (1, 1, (0, 1), "all_gather_v", 3, (6, 6)),
        (1, 1, (2, 3), "all_gather_v", 3, (6, 6)),
    ]


def test_ledger_independent_of_workers():
    rng = np.random.default_rng(5)
    payloads = [rng.standard_normal((2, 3)) for _ in range(4)]
    ledgers = [run_world(4, _mixed_program(payloads, 4), workers=w)[0].ledger for w in (1, 2, None)]
    assert ledgers[0] == ledgers[1] == ledgers[2]


def test_repeated_run_appends_deterministically():
    def program(ctx):
        return ctx.all_reduce((0, 1), torch.ones(2, dtype=torch.float64), "sum")

    world = SimWorld(2, device="cpu")
    world.run(program)
    world.run(program)
    assert len(world.ledger) == 2
    assert world.ledger[0].epoch == 1 and world.ledger[1].epoch == 2


@pytest.mark.parametrize("counts", [[[0, 3], [2, 1]], [[1, 1], [1, 1]], [[3, 0], [0, 2]]])
def test_a2a_ledger_excludes_self_traffic(counts):
    counts = np.array(counts)

    def program(ctx):
        r = rows(np.full((int(counts[ctx.rank].sum()), 2), float(ctx.rank)))
        return ctx.all_to_all_v((0, 1), VarBuffer.from_rows(r, counts[ctx.rank]))

    world, res = run_world(2, program)
    assert counts.sum() == sum(int(r.counts.sum()) for r in res)
    assert world.ledger[0].total_elements == (counts.sum() - np.trace(counts)) * 2


def test_exchange_meta_takes_a_round_but_no_record():
    def program(ctx):
        ctx.exchange_meta((0, 1), ctx.rank)
        ctx.all_gather_v((0, 1), VarBuffer.from_rows(rows(np.zeros((1, 4)))))

    world, _ = run_world(2, program)
    (rec,) = world.ledger
    assert rec.seq == 1 and rec.primitive == "all_gather_v"


def test_reduce_scatter_charges_non_owned_partitions():
    def program(ctx):
        return ctx.reduce_scatter_v((0, 1, 2), torch.ones(6 * 2, dtype=torch.float64), [1, 2, 3], 2)

    world, res = run_world(3, program)
    assert [int(r.shape[0]) for r in res] == [1, 2, 3]
    assert world.ledger[0].elements_sent == (10, 8, 6)


def test_traffic_stats_spans():
    world = SimWorld(2, device="cpu")
    assert traffic_stats(world, ClusterModel()).total_bytes == 0.0

    def gather(ctx):
        ctx.all_gather_v((0, 1), VarBuffer.from_rows(rows(np.zeros((1, 4)))))

    world, _ = run_world(2, gather)
    stats = traffic_stats(world, ClusterModel(node_size=8))
    assert stats.bytes_for("all_gather_v", "intra") == 2 * 4 * 8
    assert stats.bytes_for("all_gather_v", "inter") == 0.0

    def a2a(ctx):
        if ctx.rank in (0, 8):
            ctx.all_to_all_v((0, 8), VarBuffer.from_rows(rows(np.zeros((2, 4))), [1, 1]))

    world, _ = run_world(9, a2a)
    stats = traffic_stats(world, ClusterModel(node_size=8), elem_bytes=2.0)
    assert stats.bytes_for("all_to_all_v", "inter") == 2 * 4 * 2
    assert stats.bytes_for("all_to_all_v", "intra") == 0.0


def test_account_rejects_mismatched_primitives():
    def program(ctx):
        ctx.account((0, 1), "all_gather_v" if ctx.rank == 0 else "all_reduce", 1, 1)

    world = SimWorld(2, device="cpu")
    with pytest.raises(ProtocolError):
        world.run(program)

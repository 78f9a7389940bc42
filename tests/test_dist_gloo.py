"""World-size-2 (and 3) torch.distributed tests on CPU with the gloo backend.

They exercise the production multi-process path (NcclWorld/NcclRankContext:
process groups for the folded meshes, count all-gather, batched P2P, the
-V collectives) on CPU tensors, against the reference's collective semantics
(/root/reference/pkg/tests/test_collectives.py cases restated)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        res = globals()[fn_name](rank, world)
        q.put((rank, "ok", res))
    except BaseException as exc:  # noqa: BLE001
        import traceback

        q.put((rank, "err", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _run(fn_name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, status, res = q.get(timeout=120)
        assert status == "ok", res
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
    return out


# ---------------------------------------------------------------- programs
def prog_a2a_definition(rank, world):
    from paper_2504_14960_b200.collectives import NcclWorld, NcclRankContext, VarBuffer

    w = NcclWorld()
    ctx = NcclRankContext(w)
    vals = [1.0, 2.0] if rank == 0 else [3.0, 4.0]
    send = torch.tensor([[vals[0], vals[0]], [vals[1], vals[1]]])
    out = ctx.all_to_all_v((0, 1), VarBuffer.from_rows(send, [1, 1]))
    # ragged: r0 counts [0, 2], r1 counts [1, 0]
    if rank == 0:
        s2 = VarBuffer.from_rows(torch.ones((2, 4)), [0, 2])
    else:
        s2 = VarBuffer.from_rows(torch.full((1, 4), 7.0), [1, 0])
    o2 = ctx.all_to_all_v((0, 1), s2)
    return out.rows().tolist(), o2.rows().tolist(), o2.counts.tolist()


def prog_a2a_double_apply(rank, world):
    from paper_2504_14960_b200.collectives import NcclWorld, NcclRankContext, VarBuffer

    ctx = NcclRankContext(NcclWorld())
    rng = np.random.default_rng(3)
    counts = rng.integers(0, 4, size=(world, world))
    payloads = [rng.standard_normal((int(counts[r].sum()), 3)) for r in range(world)]
    group = tuple(range(world))
    mine = torch.as_tensor(payloads[rank])
    out = ctx.all_to_all_v(group, VarBuffer.from_rows(mine, counts[rank]))
    back = ctx.all_to_all_v(group, VarBuffer(out.values, 3, out.counts))
    return bool(torch.equal(back.rows(), mine))


def prog_gather_reduce(rank, world):
    from paper_2504_14960_b200.collectives import NcclWorld, NcclRankContext, VarBuffer

    ctx = NcclRankContext(NcclWorld())
    group = tuple(range(world))
    mine = torch.full((rank + 1, 2), float(rank))
    buf, counts = ctx.all_gather_v(group, VarBuffer.from_rows(mine))
    vals = torch.arange(12.0).reshape(6, 2) * (rank + 1)
    rs = ctx.reduce_scatter_v(group, vals, [2, 4] if world == 2 else [2, 2, 2], 2)
    ar = ctx.all_reduce(group, torch.tensor([1.0, float(rank)]), "sum")
    meta = ctx.exchange_meta(group, {"r": rank})
    return buf.rows().tolist(), counts.tolist(), rs.tolist(), ar.tolist(), meta


def prog_layer_exchange(rank, world):
    """The layer's count exchange + all_to_all_single of the padded
    per-expert layout: (sender, local expert) segments land aligned."""
    from paper_2504_14960_b200.collectives import NcclWorld, NcclRankContext
    from paper_2504_14960_b200.dispatcher import exchange_plan

    nw = NcclWorld()
    nw.setup_groups([[tuple(range(world))]])
    ctx = NcclRankContext(nw)
    L_, A = 2, 4
    E = world * L_
    rng = np.random.default_rng(100 + rank)
    counts = rng.integers(0, 7, size=E)  # my kept pairs per global expert
    all_counts = ctx.gather_counts(tuple(range(world)), torch.as_tensor(counts))
    xp = exchange_plan(all_counts, rank, L_, None, align=A)
    # padded send layout; rows carry (src rank, global expert, ordinal), pads = -1
    send = []
    for e in range(E):
        send += [[rank, e, i] for i in range(counts[e])]
        send += [[-1, -1, -1]] * int((-counts[e]) % A)
    send = torch.tensor(send, dtype=torch.float32).reshape(-1, 3)
    recv = torch.full((sum(xp.recv_splits), 3), -2.0)
    ctx.a2a_single(tuple(range(world)), send, xp.send_splits, recv, xp.recv_splits)
    return all_counts.tolist(), recv.tolist(), xp.group_off, xp.group_expert


# ---------------------------------------------------------------- tests
def test_all_to_all_v_definition_and_ragged():
    out = _run("prog_a2a_definition")
    assert out[0][0] == [[1.0, 1.0], [3.0, 3.0]]
    assert out[1][0] == [[2.0, 2.0], [4.0, 4.0]]
    assert out[0][2] == [0, 1] and out[1][2] == [2, 0]
    assert out[0][1] == [[7.0] * 4]
    assert out[1][1] == [[1.0] * 4] * 2


@pytest.mark.parametrize("world", [2, 3])
def test_all_to_all_v_double_apply_restores(world):
    out = _run("prog_a2a_double_apply", world)
    assert all(out.values())


def test_all_gather_reduce_scatter_all_reduce():
    out = _run("prog_gather_reduce")
    for r in range(2):
        rows, counts, rs, ar, meta = out[r]
        assert rows == [[0.0, 0.0], [1.0, 1.0], [1.0, 1.0]]
        assert counts == [1, 2]
        assert ar == [2.0, 1.0]
        assert meta == {0: {"r": 0}, 1: {"r": 1}}
    full = (np.arange(12.0).reshape(6, 2) * 3).tolist()  # (1 + 2) * values, folded over ranks
    assert out[0][2] == full[:2] and out[1][2] == full[2:]


@pytest.mark.parametrize("world", [2, 3])
def test_layer_exchange_lands_aligned_sender_expert_segments(world):
    out = _run("prog_layer_exchange", world)
    L_ = 2
    counts = np.array(out[0][0])
    for me in range(world):
        _, recv, goff, gexp = out[me]
        recv = np.array(recv)
        assert goff[-1] == recv.shape[0]
        g = 0
        for s in range(world):
            for le in range(L_):
                e = me * L_ + le
                assert gexp[g] == le and goff[g] % 4 == 0
                seg = recv[goff[g]:goff[g + 1]]
                want = [[s, e, i] for i in range(counts[s, e])]
                assert seg[:len(want)].tolist() == want, (me, s, le)
                assert (seg[len(want):] == -1).all()
                g += 1

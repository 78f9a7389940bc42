"""Host-side logic on CPU: topology/group generation and token partition vs
reference golden data, exchange-layout arithmetic, the C-ABI library's
exported symbols, and API validation errors (no GPU compute)."""
import ctypes
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2504_14960_b200 import _lib, errors
from paper_2504_14960_b200.dispatcher import exchange_plan, token_partition
from paper_2504_14960_b200.topology import (ParallelTopology, check_pp_consistency,
                                            generate_parallel_groups, sequence_group)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _golden_topology():
    with open(os.path.join(ROOT, "tests", "golden", "topology.json")) as f:
        return json.load(f)


def test_groups_match_reference():
    for case in _golden_topology():
        if "args" not in case:
            continue
        w, tp, cp, pp, ep, etp, layout = case["args"]
        topo = ParallelTopology(world_size=w, tp=tp, cp=cp, pp=pp, ep=ep, etp=etp, layout=layout)
        g = generate_parallel_groups(topo)
        assert {k: [list(x) for x in v] for k, v in g.attention.items()} == case["attention"]
        assert {k: [list(x) for x in v] for k, v in g.moe.items()} == case["moe"]
        assert [list(sequence_group(topo, r)) for r in range(w)] == case["seq"]
        assert [list(topo.attn_coords(r)) for r in range(w)] == case["attn_coords"]
        assert [list(topo.moe_coords(r)) for r in range(w)] == case["moe_coords"]


def test_token_partition_matches_reference():
    for case in _golden_topology():
        if "partition" not in case:
            continue
        tp, cp, dp = case["partition"]
        topo = ParallelTopology(world_size=tp * cp * dp, tp=tp, cp=cp, ep=1)
        parts = token_partition(topo, 16, 2 * dp)
        assert [p.tolist() for p in parts] == case["parts"]


def test_pp_consistency_flags_listing1_mismatch():
    bad = ParallelTopology(world_size=8, tp=2, cp=2, pp=2, ep=2, etp=1, layout="listing1")
    assert not check_pp_consistency(generate_parallel_groups(bad)).consistent
    good = ParallelTopology(world_size=8, tp=2, cp=2, pp=2, ep=2, etp=1)
    assert check_pp_consistency(generate_parallel_groups(good)).consistent


def test_topology_validation_errors():
    with pytest.raises(errors.ValidationError) as e:
        ParallelTopology(world_size=6, tp=4)
    assert e.value.constraint == "tp|world_size"
    with pytest.raises(errors.ValidationError):
        token_partition(ParallelTopology(world_size=4, tp=4), seq_len=6, batch=1)


def test_exchange_plan_arithmetic():
    # EP group of 2, L=2 local experts: member s's counts over 4 global experts
    counts = np.array([[3, 1, 2, 0], [1, 4, 0, 5]])
    xp = exchange_plan(counts, 1, 2, None, align=4)
    # rank at EP position 1 (experts 2, 3) sends its padded chunks: to 0 -> pad(1)+pad(4) = 4+4,
    # to itself -> pad(0)+pad(5) = 0+8
    assert xp.send_splits == [8, 8]
    # receives from 0: pad(2)+pad(0) = 4, from 1: pad(0)+pad(5) = 8
    assert xp.recv_splits == [4, 8]
    np.testing.assert_array_equal(xp.recv_counts, [[2, 0], [0, 5]])
    assert xp.group_off == [0, 4, 4, 4, 12]
    assert xp.group_expert == [0, 1, 0, 1]
    # ETP of 2: member blocks concatenated, groups member-major
    xp2 = exchange_plan(counts, 1, 2, np.array([[4, 0, 0, 8], [8, 4, 0, 0]]), align=4)
    assert xp2.block_off.tolist() == [0, 12, 24]
    assert xp2.group_off == [0, 4, 4, 4, 12, 20, 24, 24, 24]
    assert xp2.group_expert == [0, 1, 0, 1, 0, 1, 0, 1]


def test_library_exports_every_declared_symbol():
    """The C ABI in include/b200moe.h is what libb200moe.so exports (no GPU calls)."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libb200moe.so not built")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    hdr = open(os.path.join(ROOT, "include", "b200moe.h")).read()
    import re

    declared = sorted(set(re.findall(r"B200MOE_API [^;(]*?\b(b200moe_\w+)\s*\(", hdr)))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_lib.exported_symbols()) <= set(declared)
    assert lib.b200moe_version  # callable without a device
    lib.b200moe_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.b200moe_version()


def test_library_is_sm100a_only():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libb200moe.so not built")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout


def test_no_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libb200moe.so not built")
    with pytest.raises(RuntimeError):
        _lib.load()


def test_peer_exchange_wire_rows_match_reference_ledger(golden):
    """The device exchange moves exactly the token rows the reference's
    collectives charge on the wire (SimWorld ledger: all_to_all_v +
    all_gather_v + reduce_scatter_v), for every golden multi-rank topology."""
    from paper_2504_14960_b200.peer import wire_rows

    d = golden("layer")
    checked = 0
    for c in sorted({k.split("_")[0] for k in d if k.startswith("l")}):
        w, tp, cp, ep, etp = (int(v) for v in d[c + "_meta"][:5])
        if w == 1:
            continue
        topo = ParallelTopology(world_size=w, tp=tp, cp=cp, ep=ep, etp=etp)
        counts = [d[c + f"_counts{r}"] for r in range(w)]
        assert wire_rows(counts, topo) == int(d[c + "_ledger_rows"].sum()), c
        checked += 1
    assert checked >= 4

"""World-size-2 gloo tests (CPU) of the KV-head sharding host logic: the shard
plan, the gate-bank rows each rank takes, and the head-output all-gather that
reassembles engine.cpp's [T][Hq*d] layout.  The same code runs over NCCL on
B200s in bench.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_17452_b200.sharding import gather_heads, shard_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q_heads, kv_heads, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = shard_plan(q_heads, kv_heads, world, rank)
        B, T, d = 2, 5, 8
        # reference output: value encodes (b, t, global q head, c)
        full = torch.arange(B * T * q_heads * d, dtype=torch.float32).reshape(B, T, q_heads, d)
        local = full[:, :, sh.q_head_offset: sh.q_head_offset + sh.q_heads].contiguous()
        got = gather_heads(local, world)
        ok = torch.equal(got, full)
        # decode-shaped outputs [B][Hq][d]
        dfull = full[:, 0]
        dloc = dfull[:, sh.q_head_offset: sh.q_head_offset + sh.q_heads].contiguous()
        ok = ok and torch.equal(gather_heads(dloc, world), dfull)
        # each rank's q heads belong to its own kv heads (GQA group never straddles)
        gs = q_heads // kv_heads
        owners = {(sh.q_head_offset + j) // gs for j in range(sh.q_heads)}
        ok = ok and owners == set(range(sh.kv_head_offset, sh.kv_head_offset + sh.kv_heads))
        ret[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q_heads,kv_heads", [(32, 8), (8, 2)])
def test_gather_heads_world2(q_heads, kv_heads):
    mgr = mp.Manager()
    ret = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, q_heads, kv_heads, ret), nprocs=2, join=True)
    assert ret[0] and ret[1]


def test_shard_plan_partitions_heads():
    for world in (1, 2, 4, 8):
        seen_kv, seen_q = [], []
        for r in range(world):
            sh = shard_plan(32, 8, world, r)
            seen_kv += list(range(sh.kv_head_offset, sh.kv_head_offset + sh.kv_heads))
            seen_q += list(range(sh.q_head_offset, sh.q_head_offset + sh.q_heads))
        assert seen_kv == list(range(8)) and seen_q == list(range(32))
    with pytest.raises(ValueError):
        shard_plan(32, 8, 3, 0)


def test_sharded_gate_rows_match_unsharded(orc):
    """The bank rows a shard takes (kv_head_offset) equal the unsharded rows:
    the per-rank oracle session reproduces the full session's per-head gates."""
    import oracle as O

    L, Hq, Hkv, d, T, W = 1, 8, 4, 16, 40, 8
    bank = orc.gate_random_init(L, Hkv, d, d, 17, 0.5, -2.5)
    x = orc.gaussian(18, T * (Hq + 2 * Hkv) * d)
    q = x[: T * Hq * d].reshape(T, Hq, d)
    k = x[T * Hq * d: T * (Hq + Hkv) * d].reshape(T, Hkv, d)
    v = x[T * (Hq + Hkv) * d:].reshape(T, Hkv, d)
    full = O.Session(orc, L, Hq, Hkv, d, d, W, gate_bank=bank, max_tokens=T)
    fo, fg, fb, _ = full.prefill_layer(0, q, k, v)
    outs = []
    for r in range(2):
        sh = shard_plan(Hq, Hkv, 2, r)
        kv = slice(sh.kv_head_offset, sh.kv_head_offset + sh.kv_heads)
        qs = slice(sh.q_head_offset, sh.q_head_offset + sh.q_heads)
        s = O.Session(orc, L, sh.q_heads, sh.kv_heads, d, d, W, gate_bank=np.ascontiguousarray(bank[:, kv]),
                      max_tokens=T)
        o, g, b, _ = s.prefill_layer(0, np.ascontiguousarray(q[:, qs]), np.ascontiguousarray(k[:, kv]),
                                     np.ascontiguousarray(v[:, kv]))
        assert np.array_equal(g, fg[kv]) and np.array_equal(b, fb[kv])
        outs.append(o)
    assert np.array_equal(np.concatenate(outs, axis=1), fo)  # sharding is bitwise neutral

"""C1 over peer memory (wgkv_peer_*, comm.cuh): the decode-sized head
all-gather as LL words {data, flag} stored straight into every rank's exchange
region -- from inside the decode layer's merge (wgkv_peer_decode) or by a push
kernel -- and unpacked by a reader that polls the words.

One GPU hosts a world of one for real (the region opened through its own IPC
handle) and N "virtual" ranks whose regions all live on this GPU: every rank's
layer m runs before any rank's layer m + 1 (which unpacks exchange m), so no
kernel ever waits on one enqueued after it.  The unpacked results must equal
the unsharded context's decode output BITWISE (the reference's concat
layout, engine.cpp:234-238).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def W():
    import paper_2512_17452_b200 as W_

    W_.load()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return W_


def test_peer_world_one(W, orc):
    """A world of one through the real path: wgkv_peer_alloc (cudaMalloc +
    cudaIpcMemHandle) + wgkv_peer_open; push + unpack, rows below max_rows,
    more exchanges than slots; the result views follow each exchange."""
    hq, hkv, d, B = 8, 2, 128, 4
    s = W.Session(1, hq, hkv, d, d, 64, max_seqs=B, max_tokens=64, gate_bank=orc.gate_random_init(1, hkv, d, d, 3))
    h = s.peer_alloc(1, B)
    assert len(h) == 64
    s.peer_open(1, 0, [h])
    xs = []
    for i, rows in enumerate((4, 3, 1, 4, 2, 4, 4)):
        x = torch.randn(rows, hq, d, device="cuda").to(torch.bfloat16)
        got = s.peer_allgather_heads(x, wait=True)
        s.sync()
        assert torch.equal(got, x), i
        xs.append(x)
    for back in range(4):  # the last four exchanges stay readable
        assert torch.equal(s.peer_result(back, xs[-1 - back].shape[0]), xs[-1 - back]), back
    # pending exchanges: unpacked in order by the next exchange or by peer_wait
    a, b = (torch.randn(B, hq, d, device="cuda").to(torch.bfloat16) for _ in range(2))
    s.peer_allgather_heads(a, wait=False)
    s.peer_allgather_heads(b, wait=False)
    s.peer_wait()
    s.sync()
    assert torch.equal(s.peer_result(1, B), a) and torch.equal(s.peer_result(0, B), b)


def _decode_inputs(seed, L, B, T, hq, hkv, d, steps):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    rnd = lambda *sh: torch.randn(*sh, device="cuda", generator=gen).to(torch.bfloat16)  # noqa: E731
    return (rnd(L, B, T, hq, d), rnd(L, B, T, hkv, d), rnd(L, B, T, hkv, d),
            rnd(steps, L, B, hq, d), rnd(steps, L, B, hkv, d), rnd(steps, L, B, hkv, d))


@pytest.mark.parametrize("N,B", [(2, 2), (4, 2), (8, 4), (2, 8)])
def test_peer_virtual_shards_decode(W, orc, N, B):
    """N contexts (kv_head_offset = r * 8 / N) on one GPU with wgkv_peer_decode:
    each decode layer pushes its rows into all N regions from inside its merge
    (the fused single-kernel layer for few pairs, the finish kernel otherwise)
    and unpacks the previous layer's exchange in one of its CTAs.  Every
    rank's result of every exchange equals the unsharded decode output
    bitwise (K5's split pinned), over several steps x two layers (more
    exchanges than slots)."""
    T, hq, hkv, d, Wn, steps, L = 700, 32, 8, 128, 128, 3, 2
    q, k, v, qd, kd, vd = _decode_inputs(5, L, B, T, hq, hkv, d, steps)
    bank = orc.gate_random_init(L, hkv, d, d, 31, 0.1, -2.0)

    def session(hqs, hks, off, pin):
        return W.Session(L, hqs, hks, d, d, Wn, rope_base=5e5, max_seqs=B, max_tokens=T + steps, gate_bank=bank,
                         kv_head_offset=off, decode_chunk_pages=pin)

    hk, hqs = hkv // N, hq // N
    pin = 16 if hk * B > 8 else 0  # few pairs: the fused layer (unpinned); its split follows the pairs only
    full = [session(hqs, hk, r * hk, pin) for r in range(N)]  # per-shard references, no exchange
    parts = [session(hqs, hk, r * hk, pin) for r in range(N)]
    nbytes = parts[0].peer_region_bytes(N, B)
    regions = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(N)]
    sl = lambda x, r, w: x[..., r * w:(r + 1) * w, :].contiguous()  # noqa: E731
    for r in range(N):
        parts[r].peer_attach(N, r, B, regions)
        parts[r].peer_decode(True)
        for s_ in (full[r], parts[r]):
            for l in range(L):
                s_.prefill_layer(l, sl(q[l], r, hqs), sl(k[l], r, hk), sl(v[l], r, hk))
    want = []
    for i in range(steps):
        for l in range(L):
            outs = []
            for r in range(N):
                a = (sl(qd[i, l], r, hqs), sl(kd[i, l], r, hk), sl(vd[i, l], r, hk))
                outs.append(full[r].decode_layer(l, *a).clone())
                got = parts[r].decode_layer(l, *a)
                torch.cuda.synchronize()
                assert torch.equal(got, outs[-1]), (N, i, l, r)  # the exchange does not perturb the layer
            want.append(torch.cat(outs, dim=1))
            if len(want) >= 2:  # exchange e - 1 was unpacked by every rank's layer e
                for r in range(N):
                    assert torch.equal(parts[r].peer_result(1, B), want[-2]), (N, i, l, r)
    for r in range(N):
        parts[r].peer_wait()
    torch.cuda.synchronize()
    for r in range(N):
        for back in range(4):
            assert torch.equal(parts[r].peer_result(back, B), want[-1 - back]), (N, r, back)


def test_peer_decode_in_cuda_graph(W, orc):
    """Four decode layers (the fused layer pushing, the next layer unpacking)
    and a closing wgkv_peer_wait, captured in one CUDA graph (bench.py's token
    step) and replayed: the layer outputs equal an eager session without the
    exchange bitwise, and the four results hold the four layers' outputs."""
    B, T, hq, hkv, d, Wn, steps, L = 2, 500, 8, 2, 128, 64, 3, 4
    q, k, v, qd, kd, vd = _decode_inputs(9, L, B, T, hq, hkv, d, steps)
    bank = orc.gate_random_init(L, hkv, d, d, 13, 0.1, -1.5)
    mk = lambda: W.Session(L, hq, hkv, d, d, Wn, max_seqs=B, max_tokens=T + steps, gate_bank=bank)  # noqa: E731
    b, c = mk(), mk()
    for s in (b, c):
        for l in range(L):
            s.prefill_layer(l, q[l], k[l], v[l])
    region = torch.zeros(b.peer_region_bytes(1, B), dtype=torch.uint8, device="cuda")
    b.peer_attach(1, 0, B, [region])
    b.peer_decode(True)
    sq, sk, sv = (torch.empty_like(x[0, 0]) for x in (qd, kd, vd))
    outs = [torch.empty(B, hq, d, dtype=torch.bfloat16, device="cuda") for _ in range(L)]
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    b.set_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for l in range(L):
            b.lib.wgkv_decode_layer(b.h, l, 0, B, W.api._p(sq), W.api._p(sk), W.api._p(sv), None,
                                    W.api._p(outs[l]), None, None)
        b.peer_wait()
    b.set_stream(torch.cuda.current_stream())
    torch.cuda.current_stream().wait_stream(st)
    for i in range(steps):  # every layer of a step reads the step's static inputs
        sq.copy_(qd[i, 0])
        sk.copy_(kd[i, 0])
        sv.copy_(vd[i, 0])
        g.replay()
        torch.cuda.synchronize()
        want = [c.decode_layer(l, qd[i, 0], kd[i, 0], vd[i, 0]).clone() for l in range(L)]
        c.sync()
        for l in range(L):
            assert torch.equal(outs[l], want[l]), (i, l)
            assert torch.equal(b.peer_result(L - 1 - l, B), want[l]), (i, l)


def test_peer_topk_decode(W, orc):
    """The non-deferred decode paths (top-k here) exchange through a push
    kernel behind the layer: same results as the layer's own output."""
    B, T, hq, hkv, d, Wn, steps, L = 2, 900, 8, 2, 128, 64, 2, 2
    q, k, v, qd, kd, vd = _decode_inputs(11, L, B, T, hq, hkv, d, steps)
    s = W.Session(L, hq, hkv, d, d, Wn, max_seqs=B, max_tokens=T + steps, topk_budget=8,
                  gate_bank=orc.gate_random_init(L, hkv, d, d, 17, 0.1, -1.5))
    for l in range(L):
        s.prefill_layer(l, q[l], k[l], v[l])
    region = torch.zeros(s.peer_region_bytes(1, B), dtype=torch.uint8, device="cuda")
    s.peer_attach(1, 0, B, [region])
    s.peer_decode(True)
    got = []
    for i in range(steps):
        for l in range(L):
            got.append(s.decode_layer(l, qd[i, l], kd[i, l], vd[i, l]).clone())
    s.peer_wait()
    s.sync()
    for back in range(4):
        assert torch.equal(s.peer_result(back, B), got[-1 - back]), back


@pytest.mark.parametrize("N", [2, 4])
def test_peer_prefill_virtual_shards(W, orc, N):
    """C1 fused into K3 (wgkv_peer_prefill): each virtual rank's tcgen05
    epilogue stores its output rows into all N regions' bulk slots; after every
    rank's layer each region's bulk slot equals the unsharded context's prefill
    output BITWISE (the reference's concat layout), for two layers (both bulk
    slots), and the layer outputs are unchanged by the exchange.  wait_ranks =
    1: a virtual rank only awaits rank 0's signal, which precedes it on the
    stream (no kernel waits on one enqueued after it)."""
    B, T, hq, hkv, d, Wn, L = 2, 1000, 32, 8, 128, 256, 2
    q, k, v, _, _, _ = _decode_inputs(21, L, B, T, hq, hkv, d, 1)
    bank = orc.gate_random_init(L, hkv, d, d, 23, 0.1, -2.0)
    mk = lambda hqs, hks, off: W.Session(L, hqs, hks, d, d, Wn, max_seqs=B, max_tokens=T,  # noqa: E731
                                         gate_bank=bank, kv_head_offset=off, attn_impl=W.ATTN_TCGEN05)
    full = mk(hq, hkv, 0)
    ref = [full.prefill_layer(l, q[l], k[l], v[l]).clone() for l in range(L)]
    full.sync()
    hk, hqs = hkv // N, hq // N
    parts = [mk(hqs, hk, r * hk) for r in range(N)]
    nbytes = parts[0].peer_region_bytes(N, B, B * T)
    regions = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(N)]
    sl = lambda x, r, w: x[..., r * w:(r + 1) * w, :].contiguous()  # noqa: E731
    for r, s in enumerate(parts):
        s.peer_attach(N, r, B, regions, wait_ranks=1, max_bulk_rows=B * T)
        s.peer_prefill(True)
    for l in range(L):
        for r, s in enumerate(parts):
            out = s.prefill_layer(l, sl(q[l], r, hqs), sl(k[l], r, hk), sl(v[l], r, hk))
            torch.cuda.synchronize()
            assert torch.equal(out, sl(ref[l], r, hqs)), (N, l, r)
        for r, s in enumerate(parts):
            got = s.peer_bulk_result(0, B * T).view(B, T, hq, d)
            assert torch.equal(got, ref[l]), (N, l, r)
    for r, s in enumerate(parts):  # the previous layer's slot is intact
        assert torch.equal(s.peer_bulk_result(1, B * T).view(B, T, hq, d), ref[L - 2]), (N, r)


def test_peer_argument_errors(W, orc):
    hq, hkv, d, B = 8, 2, 128, 2
    s = W.Session(1, hq, hkv, d, d, 64, max_seqs=B, max_tokens=64, gate_bank=orc.gate_random_init(1, hkv, d, d, 3))
    x = torch.zeros(B, hq, d, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(W._lib.LifecycleError):  # nothing attached
        s.peer_allgather_heads(x)
    with pytest.raises(W._lib.LifecycleError):
        s.peer_decode(True)
    reg, reg1 = (torch.zeros(s.peer_region_bytes(2, B), dtype=torch.uint8, device="cuda") for _ in range(2))
    with pytest.raises(ValueError):  # rank outside the world
        s.peer_attach(2, 2, B, [reg, reg1])
    with pytest.raises(ValueError):  # more awaited ranks than the world
        s.peer_attach(2, 0, B, [reg, reg1], wait_ranks=3)
    s.peer_attach(2, 0, B, [reg, reg1], wait_ranks=1)  # rank 1 emulated: only rank 0's words awaited
    with pytest.raises(W._lib.LifecycleError):  # attached twice
        s.peer_attach(2, 0, B, [reg, reg1])
    with pytest.raises(ValueError):  # rows above max_rows
        s.peer_allgather_heads(torch.zeros(B + 1, hq, d, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(ValueError):  # no exchange yet
        s.peer_result(0, B)
    with pytest.raises(W._lib.LifecycleError):  # no bulk part attached
        s.peer_prefill(True)
    out = s.peer_allgather_heads(x + 1)
    s.sync()
    assert out.shape == (B, 2 * hq, d)
    assert torch.equal(out[:, :hq], x + 1)
    with pytest.raises(ValueError):
        W.Session(1, hq, hkv, d, d, 64, max_seqs=B, max_tokens=64).peer_region_bytes(9, B)
    with pytest.raises(W._lib.NotSupported):  # fp32 contexts: no peer exchange
        f = W.Session(1, hq, hkv, d, d, 64, max_seqs=B, max_tokens=64, dtype=W.F32)
        f.peer_attach(1, 0, B, [reg])


def _ipc_rank(rank, world, port, q):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import paper_2512_17452_b200 as W_

        dist.init_process_group("gloo", rank=rank, world_size=world)
        hq, hkv, d, B = 4, 1, 128, 3
        # the whole model's gate bank (every kv head); the shard keeps its rows
        bank = 0.02 * np.random.default_rng(7).standard_normal((1, hkv * world, d * 2 * d + 2 * d + 1))
        s = W_.Session(1, hq, hkv, d, d, 64, max_seqs=B, max_tokens=64, kv_head_offset=rank * hkv, gate_bank=bank)
        s.peer_init(world, rank, B)  # cudaIpcMemHandle exchange over gloo + cudaIpcOpenMemHandle
        xs = [torch.full((B, hq, d), float(r + 1), device="cuda").to(torch.bfloat16) +
              torch.arange(B * hq * d, device="cuda").view(B, hq, d).to(torch.bfloat16) for r in range(world)]
        for it in range(5):  # more exchanges than slots
            s.peer_allgather_heads(xs[rank] * (it + 1), wait=False)
            torch.cuda.synchronize()
            dist.barrier()  # every rank's words are in before anyone unpacks: no kernel waits on another process
            s.peer_wait()
            torch.cuda.synchronize()
            want = torch.cat([x * (it + 1) for x in xs], dim=1)
            assert torch.equal(s.peer_result(0, B), want), (rank, it)
            dist.barrier()
        q.put((rank, "ok"))
    except Exception as exc:  # reported to the parent
        q.put((rank, repr(exc)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_peer_ipc_two_processes(W):
    """wgkv_peer_alloc / wgkv_peer_open across two processes (one process per
    rank, as on an N-GPU box; here both on this GPU): the regions are mapped
    through real cudaIpcMemHandle exchanges and each rank's LL words land in
    the other's region.  Pushes complete (host barrier) before any rank
    unpacks, so no kernel ever spins on another process's kernel."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_rank, args=(r, 2, port, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p_ in ps:
        p_.join(60)
    assert res == {0: "ok", 1: "ok"}, res

"""Sequence-sharded decode (paper_2506_13059_b200/sharded.py).

CPU (gloo, world_size 2): the block partition covers every block exactly once with the final
block on the last rank, and TorchComm's all-gather returns every rank's tensor in rank order.
GPU (one device, ranks emulated in-process by LocalGroup): P-way sharded selection is identical
to the unsharded selection (union of the ranks' exact tokens and rejected clusters) and the
merged output matches the unsharded output.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2506_13059_b200.sharded import owned_blocks


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n_blocks", [1, 2, 5, 16, 17])
def test_block_partition(world, n_blocks):
    owners = [[r for r in range(world) if owned_blocks(r, world)(b, n_blocks)] for b in range(n_blocks)]
    assert all(len(o) == 1 for o in owners)
    assert owners[-1] == [world - 1]
    seq = [o[0] for o in owners[:-1]]
    assert seq == sorted(seq)  # contiguous ranges in rank order keep the global cluster id order


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2506_13059_b200.sharded import TorchComm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = TorchComm()
    t = torch.full((3, 2), float(rank + 1))
    g = comm.all_gather(t)
    q.put((rank, g.numpy().tolist()))
    dist.destroy_process_group()


def test_torch_comm_all_gather_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        g = np.array(res[r])
        assert g.shape == (2, 3, 2)
        assert np.all(g[0] == 1.0) and np.all(g[1] == 2.0)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_matches_unsharded(world):
    from paper_2506_13059_b200.core import EngineConfig, HeadLayout
    from paper_2506_13059_b200.engine import DecodeEngine
    from paper_2506_13059_b200.sharded import LocalGroup, ShardedDecodeEngine

    torch.manual_seed(7)
    lay = HeadLayout(16, 4, 128)
    cfg = EngineConfig(block_size=1024, alpha=512, local_buffer=64, token_budget=256, tokens_per_centroid=8,
                       rope_theta=1e6, seed=3)
    n_seq, ctx = 2, 5000
    k = torch.randn(n_seq, lay.num_kv_heads, ctx, 128, device="cuda")
    v = torch.randn(n_seq, lay.num_kv_heads, ctx, 128, device="cuda")
    ref = DecodeEngine(cfg, lay, n_seq, tcap=ctx + 16, dtype=torch.bfloat16, use_graphs=False)
    ref.write_tokens(k, v)
    ref.prefill()
    group = LocalGroup([ShardedDecodeEngine(cfg, lay, n_seq, ctx + 16, r, world) for r in range(world)])
    for e in group.engines:
        e.write_tokens(k, v)
    group.prefill()
    assert sum(int(e.eng.led.n_fine[0]) for e in group.engines) == int(ref.led.n_fine[0])
    for step in range(3):
        q = torch.randn(n_seq, lay.num_q_heads, 128, device="cuda")
        want = ref.attend(q).clone()
        st = ref.head_stats()
        got = group.attend(q)
        rel = ((got - want).norm(dim=-1) / want.norm(dim=-1)).max().item()
        assert rel < 2e-3, rel
        for l in range(ref.L):
            want_tok = np.sort(ref.tok[l, : st[l, 0]].cpu().numpy())
            got_tok = np.sort(np.concatenate([e.eng.tok[l, : e.eng.head_stats()[l, 0]].cpu().numpy()
                                              for e in group.engines]))
            assert np.array_equal(got_tok, want_tok), (step, l)
            n_rej = sum(int(e.eng.head_stats()[l, 1]) for e in group.engines)
            assert n_rej == st[l, 1]


def _sharded_worker(rank, world, port, q):
    """One rank of a real 2-process sequence-sharded decode (torch.distributed, gloo for the
    collectives, both processes on cuda:0): ShardedDecodeEngine.step through TorchComm, checked
    against an unsharded engine built in the same process from the same seeded data."""
    import torch.distributed as dist

    from paper_2506_13059_b200.core import EngineConfig, HeadLayout
    from paper_2506_13059_b200.engine import DecodeEngine
    from paper_2506_13059_b200.sharded import ShardedDecodeEngine, TorchComm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        lay = HeadLayout(16, 4, 128)
        cfg = EngineConfig(block_size=1024, alpha=512, local_buffer=16, token_budget=256, tokens_per_centroid=8,
                           rope_theta=1e6, seed=3)
        n_seq, ctx, steps = 2, 5000, 40
        gen = torch.Generator(device="cuda").manual_seed(11)
        k = torch.randn(n_seq, lay.num_kv_heads, ctx, 128, device="cuda", generator=gen)
        v = torch.randn(n_seq, lay.num_kv_heads, ctx, 128, device="cuda", generator=gen)
        Q = torch.randn(steps, n_seq, lay.num_q_heads, 128, device="cuda", generator=gen)
        KN = torch.randn(steps, n_seq, lay.num_kv_heads, 128, device="cuda", generator=gen)
        VN = torch.randn(steps, n_seq, lay.num_kv_heads, 128, device="cuda", generator=gen)
        ref = DecodeEngine(cfg, lay, n_seq, tcap=ctx + steps + 16, dtype=torch.bfloat16, use_graphs=False)
        ref.write_tokens(k, v)
        ref.prefill()
        se = ShardedDecodeEngine(cfg, lay, n_seq, ctx + steps + 16, rank, world)
        se.write_tokens(k, v)
        se.prefill_local()
        n_all = comm.all_gather(torch.as_tensor(se.eng.led.n_fine, dtype=torch.int64)).numpy()
        se.set_gid_offsets(n_all)
        worst, tok_bad, n_upd = 0.0, 0, 0
        for t in range(steps):
            want = ref.step(Q[t], KN[t], VN[t]).clone()
            st_ref = ref.head_stats()
            toks_ref = [np.sort(ref.tok[l, : st_ref[l, 0]].cpu().numpy()) for l in range(ref.L)]
            n_upd += ref.last_update is not None
            got = se.step(Q[t], KN[t], VN[t], comm)
            worst = max(worst, ((got - want).norm(dim=-1) / want.norm(dim=-1)).max().item())
            st = se.eng.head_stats()
            mine = [se.eng.tok[l, : st[l, 0]].cpu().numpy() for l in range(ref.L)]
            allt = comm.all_gather(torch.as_tensor(np.concatenate([np.bincount(m, minlength=ctx + steps)
                                                                   for m in mine]).astype(np.int32)))
            union = allt.sum(0).numpy().reshape(ref.L, -1)
            tok_bad += sum(int(not np.array_equal(np.flatnonzero(union[l]), toks_ref[l])) for l in range(ref.L))
        q.put((rank, worst, tok_bad, n_upd))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_two_processes_with_updates():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, worst, bad, n_upd = q.get(timeout=600)
        res[r] = (worst, bad, n_upd)
    for p in procs:
        p.join(timeout=120)
    for r, (worst, bad, n_upd) in res.items():
        assert bad == 0, (r, bad)
        assert worst < 2e-3, (r, worst)
        assert n_upd >= 2, n_upd


@pytest.mark.gpu
def test_sharded_step_graph_with_nccl_collectives():
    # the sharded step captured as ONE CUDA graph with its NCCL all-gathers (a real NCCL
    # communicator, world size 1 on the one reachable GPU): replays equal the eager step
    import torch.distributed as dist

    from paper_2506_13059_b200.core import EngineConfig, HeadLayout
    from paper_2506_13059_b200.sharded import ShardedDecodeEngine, TorchComm

    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        torch.manual_seed(11)
        lay = HeadLayout(16, 4, 128)
        cfg = EngineConfig(block_size=1024, alpha=512, local_buffer=64, token_budget=256, tokens_per_centroid=8,
                           rope_theta=1e6, seed=3)
        n_seq, ctx = 2, 4000
        se = ShardedDecodeEngine(cfg, lay, n_seq, ctx + 16, 0, 1)
        se.write_tokens(torch.randn(n_seq, lay.num_kv_heads, ctx, 128, device="cuda"),
                        torch.randn(n_seq, lay.num_kv_heads, ctx, 128, device="cuda"))
        se.prefill_local()
        se.set_gid_offsets(se.eng.led.n_fine[None])
        comm = TorchComm()
        for _ in range(3):
            q = torch.randn(n_seq, lay.num_q_heads, 128, device="cuda")
            want = se.attend(q, comm).clone()
            got = se.attend_graphed(q, comm).clone()
            assert torch.equal(got, want)
        assert se._graph is not None
    finally:
        dist.destroy_process_group()

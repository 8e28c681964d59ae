"""GPU tests of the shipped entry points beyond runtime.launch: the C-ABI
drop-in for execute_plan (ff_chain_run_plan, called through ctypes the way a
reference-side binding would) and the multi-GPU M-sharding
launcher (sharding.run_sharded) at world size 2 -- two processes on the one
GPU of the test box, gloo for the host-side collectives."""

import ctypes
import json
import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-2
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _graph(kind, act, m, n, k, l):
    from paper_2512_12949_b200 import workload as W

    d = W.DimensionSpec(m, n, k, l, 2)
    return W.build_gated_ffn(d) if kind == "gated_ffn" else W.build_standard_ffn(d, act)


def _run_plan_ctypes(graph, plan, host):
    """ff_chain_run_plan exactly as INTEGRATION.md's binding calls it: plain
    descriptors, device pointers, a zeroed workspace of ff_plan_workspace_bytes."""
    import torch

    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    lib = nat.load()
    d = graph.dims
    dev = {k: torch.from_numpy(v).cuda().to(torch.bfloat16).contiguous() for k, v in host.items()}
    e = torch.empty((d.m, d.l), dtype=torch.bfloat16, device="cuda")
    ch = runtime.chain_desc(graph)
    pd = runtime.plan_desc(plan)
    ws_bytes = lib.ff_plan_workspace_bytes(ctypes.byref(ch), ctypes.byref(pd))
    assert ws_bytes > 0, lib.ff_last_error()
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
    gated = graph.kind == "gated_ffn"
    t = nat.Tensors(dev["A"].data_ptr(), dev["B0" if gated else "B"].data_ptr(),
                    dev["B1"].data_ptr() if gated else None, dev["D"].data_ptr(), e.data_ptr())
    rc = lib.ff_chain_run_plan(ctypes.byref(ch), ctypes.byref(pd), ctypes.byref(t), ws.data_ptr(), ws_bytes,
                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0, lib.ff_last_error()
    torch.cuda.synchronize()
    return e


@pytest.mark.parametrize("name,rank", [("b200_llama1b", 0), ("b200_gpt67b", 0), ("b200_gpt2s", 0),
                                       ("b200_gpt2s", 2), ("b200_conv_c5", 0)])
def test_run_plan_c_abi_matches_oracle(name, rank):
    """Reference search plans (golden, B200 profile) through the C-ABI drop-in.  gpt2s
    rank 2 (blk_l 192) has no CTA-pair lowering: ff_chain_run_plan falls back to the
    1-CTA kernels."""
    from paper_2512_12949_b200 import workload as W
    from paper_2512_12949_b200.plan import plan_from_dict

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "search_results.json")))[name]
    g = gold["graph"]
    dims = W.DimensionSpec(g["m"], g["n"], g["k"], g["l"], 2)
    graph = W.build_gated_ffn(dims) if g["kind"] == "gated_ffn" else W.build_standard_ffn(
        dims, g["activation"], logical_m=g.get("logical_m"))
    plan = plan_from_dict(gold["result"]["top"][rank]["plan"])
    d = graph.dims
    host = {k: oracle.round_bf16(v) for k, v in oracle.make_inputs(graph.kind, d.m, d.n, d.k, d.l, seed=4).items()}
    out = _run_plan_ctypes(graph, plan, host)
    got = out.float().cpu().numpy()
    ref = oracle.dense_chain(graph.kind, graph.activation, host, bf16_intermediate=True)
    assert oracle.max_relative_error(got, ref) <= TOL


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


SHARD_CASE = ("standard_ffn", "relu", 1040, 2048, 1024, 1024)  # 1040 rows: shards of 528 / 512


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2512_12949_b200 import runtime, sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        kind, act, m, n, k, l = SHARD_CASE
        graph = _graph(kind, act, m, n, k, l)
        host = {name: oracle.round_bf16(v) for name, v in oracle.make_inputs(kind, m, n, k, l, seed=8).items()}
        dev = {name: torch.from_numpy(v).cuda().to(torch.bfloat16) for name, v in host.items()}
        mine = sharding.run_sharded(graph, dev)             # this rank's rows, real launcher
        full = sharding.run_sharded(graph, dev, gather=True)  # all-gathered E
        whole = runtime.run(graph, None, dev)                # the unsharded chain
        torch.cuda.synchronize()
        lo, hi = sharding.shard_bounds(m, world, rank)
        ref = oracle.dense_chain(kind, act, host, bf16_intermediate=True)
        err_mine = oracle.max_relative_error(mine.float().cpu().numpy(), ref[lo:hi])
        err_full = oracle.max_relative_error(full.float().cpu().numpy(), ref)
        same_rows = bool(torch.equal(full[lo:hi], mine))
        diff = oracle.max_relative_error(full.float().cpu().numpy(), whole.float().cpu().numpy())
        q.put((rank, err_mine, err_full, same_rows, diff, tuple(full.shape), None))
        dist.destroy_process_group()
    except Exception as exc:  # report, do not hang the parent
        q.put((rank, None, None, None, None, None, repr(exc)))


def test_run_sharded_world2_equals_unsharded():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, err_mine, err_full, same_rows, diff, shape, exc in results:
        assert exc is None, exc
        assert err_mine <= TOL and err_full <= TOL, (rank, err_mine, err_full)
        assert same_rows
        assert shape == (SHARD_CASE[2], SHARD_CASE[5])
        assert diff <= TOL  # sharded vs unsharded launch: same chain, other launch shapes
    assert all(p.exitcode == 0 for p in procs)

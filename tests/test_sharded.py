"""The expert-sharded layer (paper_2406_04984_b200/sharded.py) with world_size 2 over gloo on CPU: every exchange
of the protocol (dispatch, candidate return, ambiguous re-scoring round trip, union all-reduce, all-gather,
reduce-scatter) runs for real; per-rank compute is the fp64 oracle engine. Results must equal the unsharded
reference computation: indices bit for bit, values to fp64 round-off."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _inputs(T_per_rank, world, d=32, M=64, N=8, seed=3):
    b = 1 / np.sqrt(d)
    w_a = O.bf16_round(O.uniform(O.mix_seed(seed, 1), (d, M), -b, b))
    w_a[:, 1::2] = w_a[:, 0::2]  # duplicate keys: exact ties at the top-K boundary force the re-scoring exchange
    w_g = O.bf16_round(O.uniform(O.mix_seed(seed, 2), (N, d), -b, b))
    w_b = O.bf16_round(O.uniform(O.mix_seed(seed, 3), (M, d), -b, b))
    h = O.bf16_round(O.uniform(O.mix_seed(seed, 4), (T_per_rank * world, d), -1, 1))
    g = O.bf16_round(O.uniform(O.mix_seed(seed, 5), (T_per_rank * world, d), -1, 1))
    return w_a, w_b, w_g, h, g


def _worker(rank, world, port, outdir, T, kk, k, lr):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from sharded_oracle_engine import OracleEngine

    from paper_2406_04984_b200.sharded import ShardedLayer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w_a, w_b, w_g, h, g = _inputs(T, world)
        eng = OracleEngine(w_a, w_b, w_g, rank, world)
        layer = ShardedLayer(eng, w_a.shape[0], w_a.shape[1], w_g.shape[0])
        mine = slice(rank * T, (rank + 1) * T)
        res = layer.step(torch.tensor(h[mine]), torch.tensor(g[mine]), kk, k, lr)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), per_token=res["per_token"].numpy(), tau=res["tau"].numpy(),
                 unioned=res["unioned"].numpy(), out=res["out"].numpy(), grad_h=res["grad_h"].numpy(),
                 w_a=eng.store.w_a, w_b=eng.store.w_b, pair_step=eng.store.pair_step,
                 rescored=layer.last["rescored"])
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,T,kk,k", [(2, 12, 3, 5), (2, 20, 2, 9), (4, 10, 3, 7)])
def test_sharded_layer_matches_unsharded_reference(world, T, kk, k):
    lr = 1e-3
    with tempfile.TemporaryDirectory() as outdir:
        mp.start_processes(_worker, args=(world, _free_port(), outdir, T, kk, k, lr), nprocs=world, join=True,
                           start_method="spawn")
        ranks = [np.load(os.path.join(outdir, f"rank{r}.npz")) for r in range(world)]
    w_a, w_b, w_g, h, g = _inputs(T, world)
    sel = O.ke_select(h, w_g, w_a, kk, k)
    for r in range(world):
        np.testing.assert_array_equal(ranks[r]["per_token"], sel["per_token"][r * T:(r + 1) * T])
        np.testing.assert_array_equal(ranks[r]["tau"], sel["tau"][r * T:(r + 1) * T])
        np.testing.assert_array_equal(ranks[r]["unioned"], sel["unioned"])
    assert sum(int(x["rescored"]) for x in ranks) > 0  # the ambiguous round trip was exercised
    S = sel["unioned"]
    wak, wbk = O.gather_adapter(w_a, w_b, S)
    out, z, _ = O.ffn_forward(h, wak, wbk)
    gwa, gwb, gh = O.ffn_backward(g, h, z, None, wak, wbk)
    full = O.OracleStore(w_a, w_b)
    full.scatter_grads(S, gwa, gwb)
    full.sparse_adam(lr)
    M_loc = w_a.shape[1] // world
    for r in range(world):
        np.testing.assert_allclose(ranks[r]["out"], out[r * T:(r + 1) * T], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(ranks[r]["grad_h"], gh[r * T:(r + 1) * T], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(ranks[r]["w_a"], full.w_a[:, r * M_loc:(r + 1) * M_loc], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(ranks[r]["w_b"], full.w_b[r * M_loc:(r + 1) * M_loc], rtol=1e-12, atol=1e-15)
        np.testing.assert_array_equal(ranks[r]["pair_step"], full.pair_step[r * M_loc:(r + 1) * M_loc])

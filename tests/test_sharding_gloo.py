"""N > 1 host logic on CPU: world-size-2 gloo processes shard a batch of graphs, build
their union plans, and reduce their timings the way bench.py does (max over ranks)."""
import os
import socket

import numpy as np

import workloads as wl
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2408_03204_b200 as mg
    from paper_2408_03204_b200 import sharding

    L = 1 << 17
    graphs = [wl.generate_console(4 + (i * 7) % 29, 0.3, 1000 + i).arrays() for i in range(24)]
    costs = [sharding.graph_cost(t, L) for t, _ in graphs]
    shards = sharding.lpt_shards(costs, world)
    mine = shards[rank]
    t, e = sharding.union_arrays([graphs[i] for i in mine])
    rd = mg.compute_render_data(mg.to_flat(mg.Graph.from_arrays(t, e)))
    n_out = rd.buffer_rows - rd.output_begin
    # every rank sees the same assignment
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    # timing reduction as in bench.py: max over ranks
    tt = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    load = torch.tensor([sum(costs[i] for i in mine)], dtype=torch.float64)
    loads = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(loads, load)
    out[rank] = (gathered, n_out, len(mine), float(tt.item()), [float(x.item()) for x in loads],
                 rd.schedule.type_codes())
    dist.destroy_process_group()


def test_graph_sharding_two_ranks():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    g0, g1 = res[0][0], res[1][0]
    assert g0 == g1
    flat = sorted(i for s in g0 for i in s)
    assert flat == list(range(24))  # every graph exactly once
    assert res[0][1] == res[0][2] and res[1][1] == res[1][2]  # one output per member console
    assert res[0][3] == res[1][3] == 2.0  # max over ranks
    loads = res[0][4]
    assert max(loads) / min(loads) < 1.15  # LPT balance
    assert res[0][5].startswith("iecnsg")


def test_lpt_is_deterministic_and_balanced():
    from paper_2408_03204_b200 import sharding
    rng = np.random.default_rng(0)
    costs = list(rng.uniform(1, 10, size=512))
    for world in (1, 2, 4, 8):
        s = sharding.lpt_shards(costs, world)
        assert sharding.lpt_shards(costs, world) == s
        assert sorted(i for x in s for i in x) == list(range(512))
        loads = [sum(costs[i] for i in x) for x in s]
        assert max(loads) - min(loads) <= max(costs)


def _grad_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_03204_b200.training import reduce_gradients
    flat = torch.arange(6, dtype=torch.float64) * (rank + 1)
    views = {3: flat[:2].view(1, 2), 7: flat[2:3].view(1, 1), 5: flat[3:].view(1, 3)}
    n = reduce_gradients(flat, dist.group.WORLD)
    out[rank] = (n, {k: v.clone().numpy().tolist() for k, v in views.items()})
    dist.destroy_process_group()


def test_shared_parameter_gradients_all_reduced_two_ranks():
    # The optimisation config's only collective: one all-reduce of the flat gradient buffer
    # (per-type tables are views into it), averaged by the world size.
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_grad_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        n, views = res[r]
        assert n == 2
        assert views[3] == [[0.0, 3.0]] and views[7] == [[6.0]] and views[5] == [[9.0, 12.0, 15.0]]

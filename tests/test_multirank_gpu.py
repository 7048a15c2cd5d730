"""Multi-GPU path with real kernels, on the one GPU a test box has.

* G processes (mp.spawn), one rank each, all on cuda:0: every rank runs the real
  SlabSession kernels for its element slab and exchanges its interface rows with the
  product's exchange code over a gloo process group (transport="host": pinned host
  staging).  The ranks' kernels never wait on one another on the GPU -- the exchange
  is a host-side transfer -- so sharing the device is safe.
* The drop-in run_integration(RunConfig(..., devices=G)) with every slab on cuda:0
  (exchange="copy": device copies instead of NCCL, the same streams and launches).

Owned rows are compared with single-device run_integration: bitwise outside the p
received interface planes (same elements, same kernel, same order), and within the
parity criterion on the interface planes (the partial sums of the two slabs are
added after integration, a different rounding order)."""

import os
import socket

import numpy as np
import pytest

from tests.parity import assert_parity

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _check_owned(full_vals, got, plan, K, p, what):
    """full_vals: host CSR values of the single-device run; got: this slab's owned rows."""
    from oracle import oracle as O
    from paper_2207_00280_b200.distributed import plane_nnz

    ip, _ = O.pattern(3, K, p)
    N = K + p
    pr = N * N
    lo, hi = ip[plan.own_lo * pr], ip[plan.own_hi * pr]
    ref = full_vals[lo:hi]
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    n_recv = plane_nnz(3, K, p, *plan.recv_planes)
    assert got[n_recv:].tobytes() == ref[n_recv:].tobytes(), f"{what}: non-interface rows differ"
    assert_parity(got, ref, ip[plan.own_lo * pr: plan.own_hi * pr + 1] - lo, what=what,
                  config=f"multi-rank {what}", path="slabs+exchange")


def _worker(rank, world, port, K, p, op, assembly, coef_seed):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2207_00280_b200 as P
        from paper_2207_00280_b200.distributed import SlabSession, slab_plan

        q = p + 1
        coef = (np.random.default_rng(coef_seed).uniform(0.5, 1.5, size=(K**3, q**3))
                if coef_seed is not None else None)
        cfg = P.RunConfig("sumfact", "device", K, p, operator=op, coefficient=coef,
                          assembly=assembly)
        plan = slab_plan(K, p, world, rank)
        sess = SlabSession(cfg, plan, transport="host")
        got = sess.step()
        torch.cuda.synchronize()
        got = got.cpu().numpy()
        full = P.run_integration(cfg).gram.values.cpu().numpy()
        _check_owned(full, got, plan, K, p, f"G={world} rank {rank} {op}/{assembly}")
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G,K,p,op,assembly,coef", [
    (2, 12, 3, "stiffness", "owner", None), (3, 12, 3, "stiffness", "owner", None),
    (4, 16, 3, "stiffness", "owner", None), (2, 9, 2, "mass", "owner", 4),
    (2, 12, 3, "stiffness_mass", "owner", 7),
    (3, 12, 4, "stiffness_mass", "owner", 5)])
def test_ranks_exchange_over_gloo_with_device_kernels(G, K, p, op, assembly, coef):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(G, _free_port(), K, p, op, assembly, coef), nprocs=G, join=True)


@pytest.mark.parametrize("G,K,p,op,assembly", [(2, 12, 3, "stiffness", "owner"),
                                               (4, 16, 3, "stiffness", "owner"),
                                               (3, 12, 2, "mass", "separable"),
                                               (3, 12, 3, "stiffness", "classical")])
def test_run_integration_devices(G, K, p, op, assembly):
    """run_integration(RunConfig(devices=G)) -- the drop-in's multi-device entry -- with
    all G slabs on cuda:0 (exchange="copy"): the GlobalGram of the shards equals the
    single-device matrix (bitwise outside the interface planes for the assembled path)."""
    import torch

    import paper_2207_00280_b200 as P
    from paper_2207_00280_b200.distributed import slab_plan
    from oracle import oracle as O

    method = "classical" if assembly == "classical" else "sumfact"
    asm = "auto" if assembly == "classical" else assembly
    one = P.run_integration(P.RunConfig(method, "device", K, p, operator=op, assembly=asm))
    cfg = P.RunConfig(method, "device", K, p, operator=op, assembly=asm, devices=G, repetitions=2)
    res = P.run_integration(cfg, device_ids=[0] * G, exchange="copy")
    assert res.gram.shards is not None and len(res.gram.shards) == G
    assert len(res.times) == 2 and all(t > 0 for t in res.times)
    full = one.gram.values.cpu().numpy()
    got_all = res.gram.host_values()
    ip, _ = O.pattern(3, K, p)
    assert_parity(got_all, full, ip, what=f"devices={G} {assembly}",
                  config=f"run_integration devices={G}", path=f"{method}/{assembly}")
    if assembly == "owner":
        for g, shard in enumerate(res.gram.shards):
            _check_owned(full, shard.cpu().numpy(), slab_plan(K, p, G, g), K, p,
                         f"devices={G} shard {g}")
    # the lazily gathered device values and the scipy view agree with the shards
    assert torch.equal(res.gram.values.cpu(), torch.from_numpy(got_all))
    assert res.gram.matrix.nnz == ip[-1]


def test_run_integration_devices_validation():
    import paper_2207_00280_b200 as P

    import torch

    n = torch.cuda.device_count()
    cfg = P.RunConfig("sumfact", "device", 12, 3, operator="stiffness", devices=2)
    with pytest.raises(ValueError):
        P.run_integration(cfg, device_ids=[0, n])  # device n does not exist
    with pytest.raises(ValueError):
        P.run_integration(cfg, device_ids=[0, 0], exchange="nccl")  # NCCL needs distinct GPUs
    with pytest.raises(ValueError):
        P.run_integration(P.RunConfig("sumfact", "device", 6, 3, devices=4), device_ids=[0] * 4)

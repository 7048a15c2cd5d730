"""Multi-rank slab decomposition + interface-row exchange on CPU (gloo).

Each rank integrates its element slab with the oracle (test infrastructure
standing in for the device kernel, which has the same slab semantics -- see
tests/test_gpu_parity.py::test_slabs_sum_to_full), then runs the product's
exchange (paper_2207_00280_b200.distributed) over gloo; the owned rows must
equal the single-process matrix."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_00280_b200.distributed import exchange_interface, plane_nnz, slab_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("K,p,G", [(8, 3, 2), (12, 2, 4), (9, 3, 3), (64, 3, 8), (256, 3, 8),
                                   (7, 1, 7)])
def test_slab_plan_partitions_rows(K, p, G):
    N = K + p
    plans = [slab_plan(K, p, G, g) for g in range(G)]
    assert plans[0].own_lo == 0 and plans[-1].own_hi == N
    assert plans[0].el_lo == 0 and plans[-1].el_hi == K
    for a, b in zip(plans, plans[1:]):
        assert a.own_hi == b.own_lo and a.el_hi == b.el_lo
        assert a.send_planes[0] == b.recv_planes[0]
        assert a.send_planes[1] - a.send_planes[0] == b.recv_planes[1] - b.recv_planes[0]
        assert a.send_planes[1] <= b.own_hi  # interface lies inside the next rank's rows
    assert sum(plane_nnz(3, K, p, pl.own_lo, pl.own_hi) for pl in plans) == \
        plane_nnz(3, K, p, 0, N)


def test_slab_plan_rejects_thin_slabs():
    with pytest.raises(ValueError):
        slab_plan(6, 3, 4, 1)


def _worker(rank, world, port, K, p, op, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O

        plan = slab_plan(K, p, world, rank)
        N = K + p
        pr = N * N
        _, _, part = O.integrate_assemble(3, K, p, op, "sumfact",
                                          el_range=(plan.el_lo, plan.el_hi),
                                          row_range=(plan.own_lo * pr, plan.comp_hi * pr))
        values = torch.from_numpy(part.copy())
        exchange_interface(plan, values)
        ip, _, full = O.integrate_assemble(3, K, p, op, "sumfact")
        lo, hi = ip[plan.own_lo * pr], ip[plan.own_hi * pr]
        got = values[: hi - lo].numpy()
        from tests.parity import compare

        st = compare(got, full[lo:hi], ip[plan.own_lo * pr: plan.own_hi * pr + 1] - lo)
        assert st["ok"], (rank, st)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("K,p,G,op", [(6, 2, 2, "stiffness"), (9, 3, 3, "mass"),
                                      (8, 2, 2, "stiffness_mass")])
def test_gloo_interface_exchange(K, p, G, op):
    mp.spawn(_worker, args=(G, _free_port(), K, p, op, p + 1), nprocs=G, join=True)


@pytest.mark.parametrize("K,p,G,op", [(6, 2, 2, "stiffness"), (9, 3, 3, "mass"),
                                      (8, 2, 4, "stiffness_mass")])
def test_recompute_halo_elements_complete_owned_rows(K, p, G, op):
    """NCCL-free ablation: SlabPlan.recompute_elements restricted to
    the owned planes gives each rank its complete rows with no exchange (checked
    with the oracle standing in for the device kernel)."""
    from oracle import oracle as O
    from tests.parity import compare

    N = K + p
    pr = N * N
    ip, _, full = O.integrate_assemble(3, K, p, op, "sumfact")
    for g in range(G):
        plan = slab_plan(K, p, G, g)
        lo_el, hi_el = plan.recompute_elements
        assert hi_el - lo_el == plan.el_hi - plan.el_lo + (p if g > 0 else 0)
        _, _, part = O.integrate_assemble(3, K, p, op, "sumfact", el_range=(lo_el, hi_el),
                                          row_range=(plan.own_lo * pr, plan.own_hi * pr))
        lo, hi = ip[plan.own_lo * pr], ip[plan.own_hi * pr]
        st = compare(part[: hi - lo], full[lo:hi], ip[plan.own_lo * pr: plan.own_hi * pr + 1] - lo)
        assert st["ok"], (g, st)

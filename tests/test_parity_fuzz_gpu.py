"""Seeded randomized GPU parity: random grid shapes (ragged extents, 1-wide blocks,
narrow and wide blocks), random block decompositions, virtual multi-GPU
partitions, execution flags and forced tile variants, each bit-exact against the
oracle (R15).  The cases are a fixed function of the seed, so a failure is
reproducible by its test id."""
from __future__ import annotations

import numpy as np
import pytest

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

pytestmark = pytest.mark.gpu

N_CASES = 32
_VARIANTS = [None, None, None, "0", "5", "1", "3", "4", "12", "13", "14"]
_FLAGS = [0, 0, 0, J.JAC_F_NO_GRAPH, J.JAC_F_UNFUSED_PACK, J.JAC_F_FMA, J.JAC_F_NO_TMA]
_VFLAGS = [0, 0, J.JAC_F_NCCL, J.JAC_F_NO_GRAPH, J.JAC_F_UNFUSED_PACK, J.JAC_F_NO_TMA]


def make_case(seed):
    """(dims, blocks, n_gpus, flags, variant, iters) for one seed; <= ~1.5 M points."""
    rng = np.random.default_rng(7919 + seed)
    while True:
        b = [int(rng.choice([1, 1, 2, 2, 3, 4])) for _ in range(3)]
        e = []
        for _ in range(3):
            kind = rng.random()
            e.append(int(rng.integers(1, 4)) if kind < 0.15 else int(rng.integers(4, 40)) if kind < 0.55
                     else int(rng.choice([32, 63, 64, 65, 96, 128, 130])))
        dims = [b[d] * e[d] for d in range(3)]
        if dims[0] * dims[1] * dims[2] <= 1_500_000:
            break
    # virtual GPUs: a grid of GPUs dividing the block grid
    n_gpus = 1
    if rng.random() < 0.4:
        cands = []
        for n in (2, 4, 8):
            try:
                J.jac_plan(*dims, *b, n, None)  # host-only planner: does n partition the blocks?
                cands.append(n)
            except J.JacError:
                pass
        n_gpus = int(rng.choice(cands)) if cands else 1
    flags = int(rng.choice(_FLAGS))
    if n_gpus > 1:  # virtual partitions: the remote path (virtual NCCL layout included)
        flags = int(rng.choice(_VFLAGS)) | J.JAC_F_VIRTUAL_GPUS
    variant = _VARIANTS[int(rng.integers(0, len(_VARIANTS)))]
    return tuple(dims), tuple(b), n_gpus, flags, variant, int(rng.integers(1, 12))


@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_parity(monkeypatch, seed):
    dims, blocks, n_gpus, flags, variant, iters = make_case(seed)
    if variant is not None:
        monkeypatch.setenv("JAC_EXPERIMENT", "1")
        monkeypatch.setenv("JAC_VARIANT", variant)
    u0 = JI.hash_field(*dims, seed=1 + seed % 3)
    with jb.Jacobi3D(dims, blocks, n_gpus=n_gpus, flags=flags) as s:
        s.set_init(u0)
        k1 = iters // 2
        s.step(k1)
        s.step(iters - k1)
        got = s.field(u0)
    want, _ = oracle.jacobi3d_omp(u0, iters)
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, (f"case {dims} blocks {blocks} gpus {n_gpus} flags {flags:#x} variant {variant} "
                           f"iters {iters}: {bad.size} mismatches")

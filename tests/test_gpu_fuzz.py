"""96 seeded random configurations against the oracle: domain and patch sizes (ragged,
thin, odd), periodic axes, obstacle fractions and kinds, one to three moving-wall
velocities on random shell sides, both layouts and precisions, graphs on / off,
step counts odd and even, and the three exchange modes (direct stores, NCCL buffers
with or without the overlap, the fused handshake with the rank as its own peer).
Each case exercises a different mix of the sweep's uniform-wall side stores, the
bounce-back lists, the tiles' non-fluid bits, direct ghost stores between patches
and periodic self-neighbours."""
import numpy as np
import pytest

import oracle
from paper_1007_1388_b200 import inputs

pytestmark = pytest.mark.gpu

TOL = {8: 1e-12, 4: 1e-5}


def random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    splits = [int(rng.integers(1, 3)) for _ in range(3)]
    patch = [int(rng.integers(1, 24)) if rng.random() < 0.2 else int(rng.integers(3, 40)) for _ in range(3)]
    domain = tuple(p * s for p, s in zip(patch, splits))
    periodic = tuple(int(rng.random() < 0.3) for _ in range(3))
    nvel = int(rng.integers(1, 4))
    wu = rng.uniform(-0.04, 0.04, size=(nvel, 3))
    fl = np.zeros((domain[2] + 2, domain[1] + 2, domain[0] + 2), np.uint8)
    # walls on the shell of every non-periodic axis, a random kind per side
    for a in range(3):
        if periodic[a]:
            continue
        for side in (0, -1):
            idx = [slice(None)] * 3
            idx[2 - a] = side
            fl[tuple(idx)] = inputs.NOSLIP if rng.random() < 0.5 else inputs.VELOCITY0 + int(rng.integers(0, nvel))
    frac = float(rng.choice([0.0, 0.0, 0.03, 0.1]))
    kinds = (inputs.NOSLIP,) + tuple(inputs.VELOCITY0 + k for k in range(nvel))
    fl = inputs.add_obstacles(fl, frac, seed=seed, kinds=kinds)
    prec = int(rng.choice([8, 4]))
    layout = int(rng.integers(0, 2))
    steps = int(rng.integers(1, 12)) * (2 if layout else 1) + int(rng.integers(0, 2))
    graphs = int(rng.integers(0, 2))
    omega = float(rng.uniform(0.6, 1.9))
    # exchange: direct ghost stores (AUTO), every neighbour through the NCCL path with
    # the shell / interior overlap (FORCE_BUFFERS), or the fused handshake with the
    # rank as its own peer (SELF_PEER)
    exchange = int(rng.choice([0, 0, 1, 2]))
    overlap = int(rng.integers(0, 2))
    return dict(domain=domain, patch=tuple(patch), periodic=periodic, fl=fl, wu=wu, prec=prec, layout=layout,
                steps=steps, graphs=graphs, omega=omega, exchange=exchange, overlap=overlap)


@pytest.mark.parametrize("seed", range(96))
def test_random_configuration_vs_oracle(seed):
    from paper_1007_1388_b200 import lbm
    c = random_case(seed)
    f0 = inputs.noise_pdfs(c["domain"], seed=seed)
    ref = oracle.run(f0, c["fl"], c["wu"], c["omega"], c["steps"], periodic=c["periodic"],
                     nthreads=oracle.max_threads())
    L = lbm.Lattice(c["domain"], c["patch"], c["omega"], c["prec"], periodic=c["periodic"], layout=c["layout"],
                    use_graphs=c["graphs"], exchange_mode=c["exchange"], overlap=c["overlap"])
    try:
        L.set_flags(c["fl"], c["wu"])
        L.set_pdfs(f0)
        L.step(c["steps"])
        got = L.get_pdfs()
    finally:
        L.close()
    m = c["fl"][1:-1, 1:-1, 1:-1] == 0
    err = float(np.abs(got[m] - ref[m]).max()) if m.any() else 0.0
    assert err <= TOL[c["prec"]], (c["domain"], c["patch"], c["periodic"], c["prec"], c["layout"], c["steps"],
                                   c["exchange"], err)

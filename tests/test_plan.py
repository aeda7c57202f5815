"""Host-only decomposition / exchange-plan tests (lbm_plan, no GPU).

What must hold (P:209-229 Blocks and ranks; P:287-313 extract -> transport ->
insert, message sizes known a priori; P:322-337 only boundary PDFs; P:590-591
5 PDFs per face cell; D3Q19 has no corner velocities, so 1 PDF per edge cell
and no corner messages):
  * every send has a matching receive on the peer (same size and offset),
  * payload bytes per rank equal the closed form (3 n^2 5 + 3 n) s on 2x2x2,
  * emulating the plan on coded data fills exactly the ghost PDFs each
    boundary cell pulls, with the neighbour's values (periodic wrap included),
  * the same holds across real processes (gloo, world_size 2).
"""
import itertools
import os
import socket

import numpy as np
import pytest

from conftest import read_golden

Q = 19


def _lbm():
    from paper_1007_1388_b200 import lbm
    return lbm


def golden_e():
    return np.array([[int(r[1]), int(r[2]), int(r[3])] for r in read_golden("d3q19_table.txt")])


def all_plans(domain, patch, nranks, periodic=(0, 0, 0), proc_grid=(0, 0, 0), force=0, precision=8):
    lbm = _lbm()
    out = []
    for r in range(nranks):
        cfg = lbm.default_config(domain, patch, precision=precision, periodic=periodic, rank=r, nranks=nranks,
                                 proc_grid=proc_grid, exchange_mode=force)
        out.append(lbm.plan(cfg))
    return out


CONFIGS = [
    dict(domain=(8, 8, 8), patch=(4, 4, 4), nranks=8),
    dict(domain=(8, 8, 8), patch=(4, 4, 4), nranks=8, periodic=(1, 1, 1)),
    dict(domain=(12, 8, 16), patch=(4, 4, 4), nranks=4),
    dict(domain=(12, 8, 16), patch=(4, 4, 4), nranks=2, periodic=(0, 1, 1)),
    dict(domain=(6, 6, 6), patch=(3, 2, 3), nranks=1, periodic=(1, 0, 1), force=1),
    dict(domain=(8, 6, 4), patch=(4, 3, 2), nranks=2, periodic=(1, 1, 1), proc_grid=(2, 1, 1)),
    dict(domain=(8, 8, 8), patch=(8, 8, 8), nranks=1, periodic=(1, 1, 1), force=1),
]


def test_direction_set():
    """The 18 neighbour directions: 6 faces + 12 edges, no corners (D3Q19)."""
    plans = all_plans((3, 3, 3), (1, 1, 1), 1, periodic=(1, 1, 1), force=1)
    info, msgs = plans[0]
    recv = [m for m in msgs if not m["send"] and m["patch_local"] == 13]  # centre patch of 3x3x3
    dirs = sorted(m["dir"] for m in recv)
    assert len(dirs) == 18 == len(set(dirs))
    assert all(1 <= sum(abs(v) for v in d) <= 2 for d in dirs)
    assert sorted(m["nq"] for m in recv) == [1] * 12 + [5] * 6


@pytest.mark.parametrize("cfg", CONFIGS)
def test_sends_match_receives(cfg):
    plans = all_plans(**cfg)
    sends = {}
    recvs = {}
    for r, (_, msgs) in enumerate(plans):
        for m in msgs:
            key = (r, m["peer"]) if m["send"] else (m["peer"], r)
            seg = (m["patch_remote"] if m["send"] else m["patch_local"], m["dir"], m["nq"], m["cells"], m["offset"])
            (sends if m["send"] else recvs).setdefault(key, []).append(seg)
    assert sends.keys() == recvs.keys()
    for k in sends:
        assert sends[k] == recvs[k], k


def test_2x2x2_halo_bytes_closed_form():
    """Per rank on a 2x2x2 grid of n^3 patches: 3 face peers x 5 n^2 + 3 edge peers x n
    PDFs each way, 6 peers (SPEC S:239's 7 is wrong, no corners)."""
    for n, prec in ((4, 8), (6, 4)):
        plans = all_plans((2 * n,) * 3, (n,) * 3, 8, precision=prec)
        for info, msgs in plans:
            assert info["peers"] == 6
            assert info["halo_bytes_remote_per_step"] == (3 * n * n * 5 + 3 * n) * prec
            assert info["messages_remote"] == 6


def test_decomposition_defaults():
    lbm = _lbm()
    for nr, grid in ((1, (1, 1, 1)), (2, (1, 1, 2)), (4, (1, 2, 2)), (8, (2, 2, 2))):
        info, _ = lbm.plan(lbm.default_config((16, 16, 16), (8, 8, 8), rank=nr - 1, nranks=nr))
        assert tuple(info["proc_grid"]) == grid
    with pytest.raises(lbm.LbmError):
        lbm.plan(lbm.default_config((16, 16, 16), (16, 16, 16), nranks=2))  # 1 patch, 2 ranks
    # the bounce-back list packs a cell's patch into 19 bits: at most 2^19 - 1 patches per rank
    with pytest.raises(lbm.LbmError, match="too many patches per rank"):
        lbm.plan(lbm.default_config((128, 64, 64), (1, 1, 1)))


# ----------------------------------------------------------------------------- emulation
def code(gx, gy, gz, q, dom):
    return float(((gz * dom[1] + gy) * dom[0] + gx) * Q + q + 1)


def emulate(domain, patch, nranks, periodic=(0, 0, 0), proc_grid=(0, 0, 0)):
    """Run the remote plan (FORCE_BUFFERS: every neighbour through buffers) on coded
    patch arrays and return {global patch id: ghost-filled array}."""
    plans = all_plans(domain, patch, nranks, periodic, proc_grid, force=1)
    pg = [domain[a] // patch[a] for a in range(3)]
    e = golden_e()
    nx, ny, nz = patch

    def pcoord(g):
        return (g % pg[0], (g // pg[0]) % pg[1], g // (pg[0] * pg[1]))

    arrays = {}
    for g in range(pg[0] * pg[1] * pg[2]):
        o = [pcoord(g)[a] * patch[a] for a in range(3)]
        A = np.full((nz + 2, ny + 2, nx + 2, Q), np.nan)
        for z, y, x in itertools.product(range(nz), range(ny), range(nx)):
            for q in range(Q):
                A[z + 1, y + 1, x + 1, q] = code(o[0] + x, o[1] + y, o[2] + z, q, domain)
        arrays[g] = A

    def region(d, recv):
        rng = []
        for a in range(3):
            n = patch[a]
            if d[a] == 1:
                rng.append([n] if recv else [0])
            elif d[a] == -1:
                rng.append([-1] if recv else [n - 1])
            else:
                rng.append(list(range(n)))
        return rng

    def qlist(d):
        return [q for q in range(1, Q) if all(e[q, a] == -d[a] for a in range(3) if d[a] != 0)]

    buffers = {}
    for r, (_, msgs) in enumerate(plans):
        for m in msgs:
            if not m["send"]:
                continue
            buf = buffers.setdefault((r, m["peer"]), {})
            rx, ry, rz = region(m["dir"], recv=False)
            vals = [arrays[m["patch_local"]][z + 1, y + 1, x + 1, q]
                    for q in qlist(m["dir"]) for z in rz for y in ry for x in rx]
            assert len(vals) == m["nq"] * m["cells"]
            for i, v in enumerate(vals):
                buf[m["offset"] + i] = v
    for r, (_, msgs) in enumerate(plans):
        for m in msgs:
            if m["send"]:
                continue
            buf = buffers[(m["peer"], r)]
            rx, ry, rz = region(m["dir"], recv=True)
            i = 0
            for q in qlist(m["dir"]):
                for z in rz:
                    for y in ry:
                        for x in rx:
                            arrays[m["patch_local"]][z + 1, y + 1, x + 1, q] = buf[m["offset"] + i]
                            i += 1
    return arrays, pg, pcoord


@pytest.mark.parametrize("cfg", [dict(domain=(4, 4, 4), patch=(2, 2, 2), nranks=8),
                                 dict(domain=(6, 4, 4), patch=(2, 2, 2), nranks=2, periodic=(1, 0, 1)),
                                 dict(domain=(3, 2, 4), patch=(3, 2, 2), nranks=1, periodic=(1, 1, 1))])
def test_emulated_exchange_fills_every_pulled_ghost(cfg):
    """After the exchange, every PDF a fluid boundary cell pulls from a ghost cell
    (x - e_i in the ghost layer) holds the neighbour's value; nothing else is needed."""
    domain, patch = cfg["domain"], cfg["patch"]
    periodic = cfg.get("periodic", (0, 0, 0))
    arrays, pg, pcoord = emulate(**cfg)
    e = golden_e()
    for g, A in arrays.items():
        o = [pcoord(g)[a] * patch[a] for a in range(3)]
        for z, y, x in itertools.product(range(patch[2]), range(patch[1]), range(patch[0])):
            for q in range(1, Q):
                s = (x - e[q, 0], y - e[q, 1], z - e[q, 2])
                if all(0 <= s[a] < patch[a] for a in range(3)):
                    continue
                gc = [o[a] + s[a] for a in range(3)]
                inside = True
                for a in range(3):
                    if gc[a] < 0 or gc[a] >= domain[a]:
                        if periodic[a]:
                            gc[a] %= domain[a]
                        else:
                            inside = False
                v = A[s[2] + 1, s[1] + 1, s[0] + 1, q]
                if inside:
                    assert v == code(gc[0], gc[1], gc[2], q, domain), (g, (x, y, z), q)
                else:
                    assert np.isnan(v)


# ----------------------------------------------------------------------------- gloo, world_size 2
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lbm = _lbm()
        domain, patch, periodic = (8, 6, 8), (4, 3, 4), (0, 1, 1)
        cfg = lbm.default_config(domain, patch, periodic=periodic, rank=rank, nranks=world)
        info, msgs = lbm.plan(cfg)
        plans = [None] * world
        dist.all_gather_object(plans, (info, msgs))
        # transport coded payloads with gloo exactly as the plan prescribes
        e = golden_e()
        peer = 1 - rank
        send = sorted((m for m in msgs if m["send"]), key=lambda m: m["offset"])
        recv = sorted((m for m in msgs if not m["send"]), key=lambda m: m["offset"])
        n_send = sum(m["nq"] * m["cells"] for m in send)
        n_recv = sum(m["nq"] * m["cells"] for m in recv)
        sb = torch.zeros(n_send, dtype=torch.float64)
        o = [info["owned_lo"][a] for a in range(3)]
        pg = [domain[a] // patch[a] for a in range(3)]
        for m in send:
            g = m["patch_local"]
            pc = (g % pg[0], (g // pg[0]) % pg[1], g // (pg[0] * pg[1]))
            base = [pc[a] * patch[a] for a in range(3)]
            d = m["dir"]
            rng = [[0] if d[a] == 1 else ([patch[a] - 1] if d[a] == -1 else list(range(patch[a]))) for a in range(3)]
            qs = [q for q in range(1, Q) if all(e[q, a] == -d[a] for a in range(3) if d[a] != 0)]
            i = m["offset"]
            for q in qs:
                for z in rng[2]:
                    for y in rng[1]:
                        for x in rng[0]:
                            sb[i] = code(base[0] + x, base[1] + y, base[2] + z, q, domain)
                            i += 1
        rb = torch.zeros(n_recv, dtype=torch.float64)
        if rank == 0:
            dist.send(sb, peer)
            dist.recv(rb, peer)
        else:
            dist.recv(rb, peer)
            dist.send(sb, peer)
        ok = True
        for m in recv:
            g = m["patch_local"]
            pc = (g % pg[0], (g // pg[0]) % pg[1], g // (pg[0] * pg[1]))
            base = [pc[a] * patch[a] for a in range(3)]
            d = m["dir"]
            rng = [[patch[a]] if d[a] == 1 else ([-1] if d[a] == -1 else list(range(patch[a]))) for a in range(3)]
            qs = [q for q in range(1, Q) if all(e[q, a] == -d[a] for a in range(3) if d[a] != 0)]
            i = m["offset"]
            for q in qs:
                for z in rng[2]:
                    for y in rng[1]:
                        for x in rng[0]:
                            gc = [(base[0] + x) % domain[0], (base[1] + y) % domain[1], (base[2] + z) % domain[2]]
                            ok = ok and float(rb[i]) == code(gc[0], gc[1], gc[2], q, domain)
                            i += 1
        result_q.put((rank, ok, info["peers"], n_send, n_recv, o))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_exchange():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, *_ in res)
    # split along z (1x1x2); z periodic -> both face neighbours are the other rank
    assert res[0][2] == 1 and res[1][2] == 1
    assert res[0][3] == res[1][4] and res[0][4] == res[1][3]

// plan.cpp -- host-only block decomposition and static ghost-exchange plan.
//
// Paper: one Patch covering the domain is cut into a Cartesian grid of Blocks
// (here "patches"), several per process; the Block's rank decides where its
// data lives.  Communication = extraction -> transport ->
// insertion, local Blocks copied directly, remote ones through buffers, one
// message per destination process, sizes known a priori.  Only
// the boundary PDFs travel: 5 per face cell, 1 per edge cell (P:322-337,
// P:590-591).  No CUDA in this file: lbm_plan() runs it on a CPU-only host.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "lbm_internal.h"

namespace lbm {

// 18 directions: lexicographic over (dz, dy, dx) in {-1,0,1}^3, minus the
// centre and the 8 corners (checked by tests/test_plan.py).
const Dir3 kDirs[NDIR] = {
    {{0, -1, -1}}, {{-1, 0, -1}}, {{0, 0, -1}}, {{1, 0, -1}}, {{0, 1, -1}}, {{-1, -1, 0}},
    {{0, -1, 0}},  {{1, -1, 0}},  {{-1, 0, 0}}, {{1, 0, 0}},  {{-1, 1, 0}}, {{0, 1, 0}},
    {{1, 1, 0}},   {{0, -1, 1}},  {{-1, 0, 1}}, {{0, 0, 1}},  {{1, 0, 1}},  {{0, 1, 1}}};

int Decomp::patch_id(const int c[3]) const { return (c[2] * pgrid[1] + c[1]) * pgrid[0] + c[0]; }

void Decomp::patch_coord(int g, int c[3]) const
{
    c[0] = g % pgrid[0];
    c[1] = (g / pgrid[0]) % pgrid[1];
    c[2] = g / (pgrid[0] * pgrid[1]);
}

int Decomp::owner(int g) const
{
    int c[3];
    patch_coord(g, c);
    int r[3] = {c[0] / brick[0], c[1] / brick[1], c[2] / brick[2]};
    return (r[2] * proc[1] + r[1]) * proc[0] + r[0];
}

int Decomp::local_to_global(int l) const
{
    int b[3] = {l % brick[0], (l / brick[0]) % brick[1], l / (brick[0] * brick[1])};
    int c[3];
    for (int a = 0; a < 3; ++a) c[a] = coord[a] * brick[a] + b[a];
    return patch_id(c);
}

int Decomp::global_to_local(int g) const
{
    if (owner(g) != rank) return -1;
    int c[3];
    patch_coord(g, c);
    int b[3];
    for (int a = 0; a < 3; ++a) b[a] = c[a] - coord[a] * brick[a];
    return (b[2] * brick[1] + b[1]) * brick[0] + b[0];
}

static thread_local char g_msg[256];

const char *decompose(const lbm_config &cfg, Decomp &dec)
{
    std::memset(&dec, 0, sizeof(dec));
    for (int a = 0; a < 3; ++a) {
        if (cfg.domain[a] <= 0) return "domain must be > 0 on every axis";
        if (cfg.patch[a] <= 0) return "patch must be > 0 on every axis";
        if (cfg.domain[a] % cfg.patch[a] != 0) {
            std::snprintf(g_msg, sizeof g_msg, "patch[%d]=%d does not divide domain[%d]=%lld", a,
                          cfg.patch[a], a, (long long)cfg.domain[a]);
            return g_msg;
        }
        if (cfg.patch[a] > 32767) return "patch too large (at most 32767 cells per axis: 16-bit tile descriptors)";
        dec.domain[a] = cfg.domain[a];
        dec.patch[a] = cfg.patch[a];
        dec.pgrid[a] = (int)(cfg.domain[a] / cfg.patch[a]);
        dec.periodic[a] = cfg.periodic[a] ? 1 : 0;
    }
    if (!(cfg.omega > 0.0 && cfg.omega < 2.0)) return "omega must satisfy 0 < omega < 2";
    if (cfg.precision != LBM_FP32 && cfg.precision != LBM_FP64) return "precision must be LBM_FP32 (4) or LBM_FP64 (8)";
    if (cfg.nranks < 1 || cfg.rank < 0 || cfg.rank >= cfg.nranks) return "need 0 <= rank < nranks";
    if (cfg.exchange_mode != LBM_EXCHANGE_AUTO && cfg.exchange_mode != LBM_EXCHANGE_FORCE_BUFFERS &&
        cfg.exchange_mode != LBM_EXCHANGE_SELF_PEER)
        return "unknown exchange_mode";
    if (cfg.exchange_mode == LBM_EXCHANGE_SELF_PEER && cfg.nranks != 1) return "exchange_mode SELF_PEER needs nranks == 1";
    if (cfg.layout != LBM_LAYOUT_AB && cfg.layout != LBM_LAYOUT_AA) return "unknown layout";
    int pg[3] = {cfg.proc_grid[0], cfg.proc_grid[1], cfg.proc_grid[2]};
    if (pg[0] == 0 && pg[1] == 0 && pg[2] == 0) {
        // Default: split z first, then y, then x.
        switch (cfg.nranks) {
        case 1: pg[0] = 1; pg[1] = 1; pg[2] = 1; break;
        case 2: pg[0] = 1; pg[1] = 1; pg[2] = 2; break;
        case 4: pg[0] = 1; pg[1] = 2; pg[2] = 2; break;
        case 8: pg[0] = 2; pg[1] = 2; pg[2] = 2; break;
        default: pg[0] = 1; pg[1] = 1; pg[2] = cfg.nranks; break;
        }
    }
    if (pg[0] < 1 || pg[1] < 1 || pg[2] < 1 || (int64_t)pg[0] * pg[1] * pg[2] != cfg.nranks)
        return "proc_grid product must equal nranks";
    for (int a = 0; a < 3; ++a) {
        if (dec.pgrid[a] % pg[a] != 0) {
            std::snprintf(g_msg, sizeof g_msg, "patches per axis %d (%d) not divisible by proc_grid (%d)", a,
                          dec.pgrid[a], pg[a]);
            return g_msg;
        }
        dec.proc[a] = pg[a];
        dec.brick[a] = dec.pgrid[a] / pg[a];
    }
    if ((int64_t)dec.pgrid[0] * dec.pgrid[1] * dec.pgrid[2] > (1 << 24)) return "too many patches";
    dec.rank = cfg.rank;
    dec.nranks = cfg.nranks;
    dec.coord[0] = cfg.rank % pg[0];
    dec.coord[1] = (cfg.rank / pg[0]) % pg[1];
    dec.coord[2] = cfg.rank / (pg[0] * pg[1]);
    // FORCE_BUFFERS and SELF_PEER: same-rank neighbours are planned as remote
    // segments (peer = this rank)
    dec.force_buffers = cfg.exchange_mode != LBM_EXCHANGE_AUTO;
    dec.nlocal = dec.brick[0] * dec.brick[1] * dec.brick[2];
    // the bounce-back list packs a cell's patch into 19 bits (kernels.cuh bb_pos)
    if (dec.nlocal >= (1 << 19)) return "too many patches per rank (at most 524287)";
    for (int a = 0; a < 3; ++a) {
        dec.owned_lo[a] = (int64_t)dec.coord[a] * dec.brick[a] * dec.patch[a];
        dec.owned_hi[a] = dec.owned_lo[a] + (int64_t)dec.brick[a] * dec.patch[a];
    }
    return "";
}

int Decomp::local_index_on_owner(int g) const
{
    int c[3];
    patch_coord(g, c);
    int b[3];
    for (int a = 0; a < 3; ++a) b[a] = c[a] % brick[a];
    return (b[2] * brick[1] + b[1]) * brick[0] + b[0];
}

// Neighbour patch of global patch g in direction d (periodic wrap), or -1.
int neighbour(const Decomp &dec, int g, const int d[3])
{
    int c[3];
    dec.patch_coord(g, c);
    for (int a = 0; a < 3; ++a) {
        c[a] += d[a];
        if (c[a] < 0 || c[a] >= dec.pgrid[a]) {
            if (!dec.periodic[a]) return -1;
            c[a] = (c[a] + dec.pgrid[a]) % dec.pgrid[a];
        }
    }
    return dec.patch_id(c);
}

// Segment through which receiving patch `recv` gets, in its ghost layer toward
// direction index k, the PDFs its boundary cells pull from neighbour `send`.
// The pulled directions i satisfy e_i[a] = -d[a] on every axis with d[a] != 0
// (a cell x pulls f_i from x - e_i): 5 for a face, 1 for an edge.
static Seg make_seg(const Decomp &dec, int recv, int send, int k, int kind)
{
    Seg s;
    std::memset(&s, 0, sizeof s);
    s.recv_patch = recv;
    s.send_patch = send;
    s.dir = k;
    for (int a = 0; a < 3; ++a) s.d[a] = kDirs[k].d[a];
    s.cells = 1;
    for (int a = 0; a < 3; ++a) {
        int n = dec.patch[a];
        if (s.d[a] == 1) {
            // receiver ghost at n <- sender boundary at 0 (AA2: receiver boundary n-1 <- sender ghost -1)
            s.recv_lo[a] = kind == EX_AA2 ? n - 1 : n;
            s.send_lo[a] = kind == EX_AA2 ? -1 : 0;
            s.size[a] = 1;
        } else if (s.d[a] == -1) {
            s.recv_lo[a] = kind == EX_AA2 ? 0 : -1;
            s.send_lo[a] = kind == EX_AA2 ? n : n - 1;
            s.size[a] = 1;
        } else {
            s.recv_lo[a] = 0;
            s.send_lo[a] = 0;
            s.size[a] = n;
        }
        s.cells *= s.size[a];
    }
    s.nq = 0;
    const int sign = kind == EX_AA1 ? 1 : -1;
    for (int i = 0; i < Q; ++i) {
        const int e[3] = {EX(i), EY(i), EZ(i)};
        bool ok = true;
        for (int a = 0; a < 3; ++a)
            if (s.d[a] != 0 && e[a] != sign * s.d[a]) ok = false;
        if (ok && i != 0 && s.nq < 5) s.q[s.nq++] = i;
    }
    return s;
}

void build_segments(const Decomp &dec, SegLists &out, int kind)
{
    out.local.clear();
    out.send.clear();
    out.recv.clear();
    // Receives / local copies: every local patch, every direction.
    for (int l = 0; l < dec.nlocal; ++l) {
        int g = dec.local_to_global(l);
        for (int k = 0; k < NDIR; ++k) {
            int nb = neighbour(dec, g, kDirs[k].d);
            if (nb < 0) continue;
            Seg s = make_seg(dec, g, nb, k, kind);
            int own = dec.owner(nb);
            s.peer = own;
            if (own == dec.rank && !dec.force_buffers)
                out.local.push_back(s);
            else
                out.recv.push_back(s);
        }
    }
    // Sends: every local patch N and every direction s whose receiver P = N + s
    // is remote (or forced through buffers); the receiver sees N in direction -s.
    for (int l = 0; l < dec.nlocal; ++l) {
        int g = dec.local_to_global(l);
        for (int k = 0; k < NDIR; ++k) {
            int p = neighbour(dec, g, kDirs[k].d);
            if (p < 0) continue;
            int own = dec.owner(p);
            if (own == dec.rank && !dec.force_buffers) continue;
            int minus[3] = {-kDirs[k].d[0], -kDirs[k].d[1], -kDirs[k].d[2]};
            int kr = -1;
            for (int j = 0; j < NDIR; ++j)
                if (kDirs[j].d[0] == minus[0] && kDirs[j].d[1] == minus[1] && kDirs[j].d[2] == minus[2]) kr = j;
            Seg s = make_seg(dec, p, g, kr, kind);
            s.peer = own;
            out.send.push_back(s);
        }
    }
    auto key = [](const Seg &a, const Seg &b) {
        if (a.peer != b.peer) return a.peer < b.peer;
        if (a.recv_patch != b.recv_patch) return a.recv_patch < b.recv_patch;
        return a.dir < b.dir;
    };
    std::sort(out.send.begin(), out.send.end(), key);
    std::sort(out.recv.begin(), out.recv.end(), key);
    for (std::vector<Seg> *v : {&out.send, &out.recv}) {
        int peer = -1;
        int64_t off = 0;
        for (Seg &s : *v) {
            if (s.peer != peer) {
                peer = s.peer;
                off = 0;
            }
            s.offset = off;
            off += (int64_t)s.nq * s.cells;
        }
    }
}

}  // namespace lbm

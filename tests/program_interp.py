"""TEST-ONLY numpy interpreter of the compiled device step program (include/owqs_host.h).

It executes the steps exactly as the kernels define them (ops on slots, decisions in the pass
prologue, reductions of the step output, grow / shrink), so that the host scheduler + compiler
can be checked against the oracle on a machine without a GPU. It is not a product path (the
product has no CPU fallback) and it shares no code with the oracle.
"""
from __future__ import annotations

import math

import numpy as np

OP_DIAG_E, OP_DIAG_Z, OP_X, OP_BFLY = 1, 2, 3, 4
ST_PASS, ST_GROW, ST_SHRINK, ST_SWAP, ST_RHOK, ST_SHRINKK = 0, 1, 2, 3, 4, 5
RED_NONE, RED_NORM, RED_RHO = 0, 1, 2


def _splitmix64(x):
    m = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def _draw(seed, ord_):
    return (_splitmix64(seed ^ _splitmix64(ord_)) >> 11) * 2.0 ** -53


class Interp:
    """rank / world / comm: sharded execution (n_global = log2(world) top positions are rank bits);
    comm provides all_reduce_sum(np.ndarray) and exchange(np.ndarray, partner) -> np.ndarray."""

    def __init__(self, prog, mode: str, seed: int = 0, forced=None, rank: int = 0, world: int = 1, comm=None):
        self.p = prog
        self.rank, self.world, self.comm = rank, world, comm
        self.ng = prog.info.get("n_global", 0)
        self.mode = {"sampled": 0, "forced": 1, "eowqs": 2}[mode]
        self.seed = seed
        K = prog.info["n_measure"]
        self.forced = np.zeros(K, np.uint8) if forced is None else np.asarray(forced, np.uint8)
        self.outcome = np.zeros(K, np.uint8)
        self.prob0 = np.zeros(K)
        self.red = np.zeros(4)
        self.err = 0

    def parity(self, off, ln, loc):
        s = 0
        for o in self.p.sig[off:off + ln]:
            s ^= loc[o] if o in loc else int(self.outcome[o])
        return s & 1

    def decide(self, m, use_red, full, loc):
        ms = self.p.mst[m]
        s = t = 0
        if self.mode != 2:
            s = self.parity(ms.s_off, ms.s_len, loc)
            t = self.parity(ms.t_off, ms.t_len, loc)
        theta = (-ms.alpha if s else ms.alpha) + (math.pi if t else 0.0)
        e = complex(math.cos(theta), -math.sin(theta))
        outc, pS, P0 = 0, 0.5, -1.0
        if self.mode != 2:
            if full:
                tot = self.red[0] + self.red[1]
                P0 = 0.5 * tot + (e * complex(self.red[2], self.red[3])).real
                P0 = min(max(P0, 0.0), tot)
                P1 = tot - P0
            else:
                nrm = self.red[0] if use_red else 1.0
                P0 = P1 = 0.5 * nrm
            outc = (0 if _draw(self.seed, ms.key) <= P0 else 1) if self.mode == 0 else int(self.forced[ms.ord]) & 1
            pS = P1 if outc else P0
            if pS < 1e-12:
                self.err = 1
                pS = 1.0
        sg = -1.0 if outc else 1.0
        if ms.reuse:
            k = (1 / math.sqrt(2)) if self.mode == 2 else 0.5 / math.sqrt(pS)
            U = np.array([[k, k * sg * e], [k, -k * sg * e]])
        else:
            k = 1.0 if self.mode == 2 else 1 / math.sqrt(2 * pS)
            U = np.array([[k, k * sg * e], [0, 0]])
        self.outcome[ms.ord] = outc
        self.prob0[ms.ord] = P0
        loc[ms.ord] = outc
        return U

    def _joint(self, d, v):
        """ST_SHRINKK: decide jk outcomes in order from rho (conditional Eq. 3 probabilities),
        project and eliminate them at once; output bit t <- position d.j_src[t]."""
        k, w = d.jk, d.width
        R = getattr(self, "rhok", None)
        R = None if R is None else R.copy()
        loc, us, pj = {}, [], 1.0
        for j in range(k):
            ms = self.p.mst[d.jm[j]]
            s = t = 0
            if self.mode != 2:
                s = self.parity(ms.s_off, ms.s_len, loc)
                t = self.parity(ms.t_off, ms.t_len, loc)
            theta = (-ms.alpha if s else ms.alpha) + (math.pi if t else 0.0)
            e = complex(math.cos(theta), -math.sin(theta))
            outc, P0 = 0, -1.0
            if self.mode != 2:
                tot = float(np.trace(R).real)
                u0 = np.array([1, e]) / math.sqrt(2)
                D = R.shape[0]
                p0 = 0.0
                for a2 in range(D // 2):
                    blk = R[2 * a2:2 * a2 + 2, 2 * a2:2 * a2 + 2]
                    p0 += (u0 @ blk @ u0.conj()).real
                p0 = min(max(p0, 0.0), tot)
                P0 = p0 / tot if tot > 0 else 0.0
                outc = (0 if _draw(self.seed, ms.key) <= P0 else 1) if self.mode == 0 else int(self.forced[ms.ord]) & 1
                pS = 1 - P0 if outc else P0
                if pS < 1e-12:
                    self.err = 1
                    pS = 1.0
                pj *= pS
                u = np.array([1, -e if outc else e]) / math.sqrt(2)
                D2 = D // 2
                Rn = np.zeros((D2, D2), dtype=complex)
                for a2 in range(D2):
                    for b2 in range(D2):
                        Rn[a2, b2] = u @ R[2 * a2:2 * a2 + 2, 2 * b2:2 * b2 + 2] @ u.conj()
                R = Rn
            sg = -1.0 if outc else 1.0
            kk = 1.0 if self.mode == 2 else 1 / math.sqrt(2)
            us.append(np.array([kk, kk * sg * e]))
            self.outcome[ms.ord] = outc
            self.prob0[ms.ord] = P0
            loc[ms.ord] = outc
        scale = 1.0 if self.mode == 2 else 1 / math.sqrt(pj)
        cv = np.array([scale * np.prod([us[j][(x >> j) & 1] for j in range(k)]) for x in range(1 << k)])
        wo = w - k
        i = np.arange(1 << wo)
        src = np.zeros_like(i)
        for tb in range(wo):
            src |= ((i >> tb) & 1) << d.j_src[tb]
        out = np.zeros(1 << wo, dtype=complex)
        for x in range(1 << k):
            off = sum(((x >> j) & 1) << d.jm_pos[j] for j in range(k))
            out += cv[x] * v[src | off]
        return out, cv

    def _allreduce(self):
        if self.world > 1:
            self.red = self.comm.all_reduce_sum(self.red.copy())

    def run(self, psi):
        """psi: the full input state (each rank takes its shard); returns the shard (world > 1)
        or the permuted output (world == 1)."""
        wl = self.p.info["phys_bits"] - self.ng
        if self.world > 1:
            st = psi[self.rank << wl:(self.rank + 1) << wl].astype(np.complex128).copy()
        else:
            st = np.zeros(2 ** self.p.info["phys_bits"], dtype=np.complex128)
            st[: psi.size] = psi
        for d in self.p.steps:
            w = d.width
            n = 1 << w
            if d.kind == 3:  # SWAP: trade the half with local bit = 1 - (rank bit) with the partner
                gb = d.swap_global - w
                b = (self.rank >> gb) & 1
                partner = self.rank ^ (1 << gb)
                idx = np.arange(n)
                half = idx[((idx >> d.swap_local) & 1) == 1 - b]
                st[half] = self.comm.exchange(st[half].copy(), partner)
                continue
            if d.kind == ST_PASS:
                loc, coefs, conds, bidx = {}, {}, {}, {}
                bi = 0
                for i in range(d.n_ops):
                    op = d.ops[i]
                    if op.type == OP_BFLY:
                        U = self.decide(op.m, bi == 0 and d.first_uses_red, False, loc)
                        if op.cond and self.parity(op.sig_off, op.sig_len, loc):
                            U = U[::-1].copy()  # folded X: swap output rows
                        coefs[i] = U
                        bidx[i] = bi
                        bi += 1
                    elif op.type != 5:
                        conds[i] = self.parity(op.sig_off, op.sig_len, loc) if op.cond else 1
                v = st[:n].copy()
                idx = np.arange(n) | (self.rank << w)  # global index (rank bits on top)
                for i in range(d.n_ops):
                    op = d.ops[i]
                    if op.type == 5:  # FLUSH: diagonals are applied directly here
                        continue
                    if op.type in (OP_DIAG_E, OP_DIAG_Z):
                        if not conds[i]:
                            continue
                        b = op.b if op.type == OP_DIAG_E else op.a
                        mask = ((idx >> op.a) & (idx >> b) & 1).astype(bool)
                        v[mask] = -v[mask]
                    else:
                        if op.type == OP_X and not conds[i]:
                            continue
                        U = coefs[i] if op.type == OP_BFLY else np.array([[0, 1], [1, 0]])
                        a = op.a
                        loc = np.arange(n)
                        i0 = loc[((loc >> a) & 1) == 0]
                        i1 = i0 | (1 << a)
                        x0, x1 = v[i0].copy(), v[i1].copy()
                        if op.type == OP_BFLY:  # absorbed CZs: x1 sign by the parity of absorb bits
                            am = d.absorb[bidx[i]]
                            par = (np.array([bin(int(j) & am).count("1") & 1 for j in idx[i1]])
                                   if am else 0)
                            x1 = x1 * (1 - 2 * par)
                        v[i0] = U[0, 0] * x0 + U[0, 1] * x1
                        v[i1] = U[1, 0] * x0 + U[1, 1] * x1
                if d.n_ops > 0:
                    st[:n] = v
                self._reduce(d, v, np.arange(n))
                for k in range(getattr(d, "n_remap", 0)):  # qubit remap at the store: swap bits a, b
                    a, b = d.remap_a[k], d.remap_b[k]
                    j = np.arange(n)
                    flip = ((j >> a) ^ (j >> b)) & 1
                    dst = j ^ (flip << a) ^ (flip << b)
                    cur = st[:n].copy()
                    st[dst] = cur
                if d.red_kind != RED_NONE:
                    self._allreduce()
            elif d.kind == ST_RHOK:  # reduced density matrix of the jk measured positions
                k = d.jk
                pos = [d.jm_pos[j] for j in range(k)]
                idx = np.arange(n)
                rest = idx[np.all([((idx >> q) & 1) == 0 for q in pos], axis=0)]
                V = np.stack([st[rest | sum(((x >> j) & 1) << pos[j] for j in range(k))] for x in range(1 << k)])
                self.rhok = V @ V.conj().T  # rho[a][b] = sum_rest v_a conj(v_b)
            elif d.kind == ST_SHRINKK:
                st_new, cv = self._joint(d, st[:n])
                m = st_new.size
                st[:m] = st_new
                if d.red_kind == RED_NORM:
                    self.red[:] = [np.vdot(st[:m], st[:m]).real, 0, 0, 0]
                    self._allreduce()
            elif d.kind == ST_GROW:
                x = st[:n] / math.sqrt(2)
                st[:n] = x
                st[n:2 * n] = x
                if d.red_kind == RED_NORM:
                    self.red[:] = [np.vdot(st[:2 * n], st[:2 * n]).real, 0, 0, 0]
                    self._allreduce()
            else:
                U = self.decide(d.shrink_m, True, bool(d.first_full_rho), {})
                b, top = d.slot, w - 1
                v = st[:n].copy()
                idx = np.arange(n)
                if b == top:
                    h = n // 2
                    st[:h] = U[0, 0] * v[:h] + U[0, 1] * v[h:]
                else:
                    r = idx[(((idx >> b) & 1) == 0) & (((idx >> top) & 1) == 0)]
                    B, T = 1 << b, 1 << top
                    st[r] = U[0, 0] * v[r] + U[0, 1] * v[r | B]
                    st[r | B] = U[0, 0] * v[r | T] + U[0, 1] * v[r | B | T]
                if d.red_kind == RED_NORM:
                    h = n // 2
                    self.red[:] = [np.vdot(st[:h], st[:h]).real, 0, 0, 0]
                    self._allreduce()
        if self.world > 1:
            return st[: 1 << wl]
        return self.permute_out(st)

    def permute_out(self, st):
        n_out = self.p.info["n_out"]
        j = np.arange(2 ** n_out)
        src = np.zeros_like(j)
        for k, s in enumerate(self.p.out_slot):
            src |= ((j >> k) & 1) << s
        return st[src]

    def _reduce(self, d, v, idx):
        if d.red_kind == RED_NORM:
            self.red[:] = [np.vdot(v, v).real, 0, 0, 0]
        elif d.red_kind == RED_RHO:
            r = d.red_slot
            b = ((idx >> r) & 1).astype(bool)
            n0 = np.vdot(v[~b], v[~b]).real
            n1 = np.vdot(v[b], v[b]).real
            i0 = idx[~b]
            c = np.vdot(v[i0], v[i0 | (1 << r)])
            self.red[:] = [n0, n1, c.real, c.imag]

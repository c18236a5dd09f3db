"""CPU restatement of the config-network generator — TEST INFRASTRUCTURE.

Specification: `paper_2110_04421_b200/confignet.py` module docstring.  This
is an independent vectorised numpy implementation of the same definition
(the CUDA one is `paper_2110_04421_b200/csrc/epi_confignet.cuh`):
  * bijections are evaluated forward over the whole domain and inverted by
    scatter (the device evaluates the inverse rounds directly), so the two
    implementations cross-check each other's inverse;
  * keyed hashes come from `oracle.rng_np` (reference rng.py:60-100 chain).
Output: a StepGraph-like triple in canonical (dst, src, kind) order.
"""

from __future__ import annotations

import numpy as np

from . import rng_np

P_RCOUNT, P_RPERM, P_WPERM, P_WSHIFT = 72, 73, 74, 75
M32 = np.uint64(0xFFFFFFFF)
GOLD32 = np.uint64(0x9E3779B1)


def radix(n):
    """b = smallest integer with b*b >= n, a = ceil(n / b) (vectorised)."""
    n = np.asarray(n, dtype=np.int64)
    b = np.ceil(np.sqrt(np.maximum(n, 1).astype(np.float64))).astype(np.int64)
    b = np.where(b * b < n, b + 1, b)
    b = np.where((b > 1) & ((b - 1) * (b - 1) >= n), b - 1, b)
    a = (n + b - 1) // b
    return a.astype(np.uint64), b.astype(np.uint64)


def _f(v, k1, k2, rad):
    h = ((v ^ k1) * k2) & M32
    h = ((h ^ (h >> np.uint64(16))) * np.uint64(0x7FEB352D)) & M32
    return ((h ^ (h >> np.uint64(15))) * rad) >> np.uint64(32)


def feistel_forward(x, k1, k2, a, b):
    """One application of the 3-round mixed-radix Feistel on [0, a*b)."""
    L, R = x // b, x % b
    L = (L + _f(R, k1[0], k2[0], a)) % a
    R = (R + _f(L, k1[1], k2[1], b)) % b
    L = (L + _f(R, k1[2], k2[2], a)) % a
    return L * b + R


def walk(x, n, k1, k2, a, b):
    """Cycle-walk the Feistel bijection until the value is < n (elementwise)."""
    out = np.asarray(x, dtype=np.uint64).copy()
    n = np.broadcast_to(np.asarray(n, dtype=np.uint64), out.shape)
    todo = np.arange(len(out))
    cur = out.copy()
    while len(todo):
        cur = feistel_forward(cur, [k[todo] if np.ndim(k) else k for k in k1],
                              [k[todo] if np.ndim(k) else k for k in k2],
                              a[todo] if np.ndim(a) else a, b[todo] if np.ndim(b) else b)
        done = cur < n[todo]
        out[todo[done]] = cur[done]
        todo, cur = todo[~done], cur[~done]
    return out.astype(np.int64)


def random_perm_keys(seed, step, slot):
    hs = [int(rng_np.hashes(seed, step, P_RPERM, [slot], r)[0]) for r in range(3)]
    return ([np.uint64(h & 0xFFFFFFFF) for h in hs],
            [np.uint64((h >> 32) | 1) for h in hs])


def random_permutation(n, seed, step, slot):
    """pi_{step,slot} as an array: pi[x] for every x in [0, n)."""
    k1, k2 = random_perm_keys(seed, step, slot)
    a, b = radix(n)
    return walk(np.arange(n, dtype=np.uint64), n, k1, k2, np.uint64(a), np.uint64(b))


def workplace_sigma(pop, seed, step):
    """For every member slot (base_w + position): the local index sigma_w(position)."""
    m_w = pop.wp_size.astype(np.int64)
    W = len(m_w)
    ha = rng_np.hashes(seed, step, P_WPERM, np.arange(W), 0)
    hb = rng_np.hashes(seed, step, P_WPERM, np.arange(W), 1)
    m16 = np.uint64(0xFFFF)
    k1 = [ha & m16, (ha >> np.uint64(32)) & m16, hb & m16]
    k2 = [((ha >> np.uint64(16)) & m16) | np.uint64(1), ((ha >> np.uint64(48)) & m16) | np.uint64(1),
          ((hb >> np.uint64(16)) & m16) | np.uint64(1)]
    owner = np.repeat(np.arange(W), m_w)
    pos = (np.arange(len(owner)) - pop.wp_base[owner]).astype(np.uint64)
    a, b = radix(m_w)
    return walk(pos, m_w[owner], [k[owner] for k in k1], [k[owner] for k in k2],
                a[owner], b[owner])


def work_shifts_all(pop, seed, step, draws):
    """r[w, j] = 1 + ((v * (m - 1)) >> 16), v = 16-bit chunk j&3 of hash (w, j>>2)."""
    W = pop.n_workplaces
    m = pop.wp_size.astype(np.uint64)
    out = np.zeros((W, draws), dtype=np.int64)
    for j in range(draws):
        h = rng_np.hashes(seed, step, P_WSHIFT, np.arange(W), j >> 2)
        v = (h >> np.uint64(16 * (j & 3))) & np.uint64(0xFFFF)
        out[:, j] = (np.uint64(1) + ((v * np.maximum(m, np.uint64(1)) - v) >> np.uint64(16))).astype(np.int64)
    return out


def random_counts(seed, step, n, table, dead):
    u = rng_np.uniforms(seed, step, P_RCOUNT, np.arange(n))
    cnt = (u[:, None] >= table[None, :]).sum(axis=1) if len(table) else np.zeros(n, np.int64)
    cnt[dead] = 0
    return cnt


def realize(pop, seed, step, dead, canonical=True):
    """All directed edges of step `step` as (src, dst, kind); canonical
    (dst, src, kind) order unless `canonical=False` (the timed CPU arm: the
    reference engine sorts the valid edges itself, engine.py:98)."""
    spec = pop.spec
    n = spec.n_agents
    dead = np.asarray(dead, dtype=bool)
    alive = ~dead
    S, D, K = [], [], []
    # households: complete graph on alive members (contiguous id ranges)
    ids = np.arange(n, dtype=np.int64)
    start = ids - pop.hh_off.astype(np.int64)
    for off in range(int(pop.hh_size.max()) if n else 0):
        c = start + off
        ok = (off < pop.hh_size) & (c != ids) & alive
        c_ok = np.where(ok, c, 0)
        ok &= alive[c_ok]
        S.append(c[ok]); D.append(ids[ok]); K.append(np.zeros(int(ok.sum()), np.int8))
    # workplaces (vectorised over all members)
    if pop.n_workplaces and spec.colleague_draws:
        base = pop.wp_base.astype(np.int64)
        m_w = pop.wp_size.astype(np.int64)
        owner = np.repeat(np.arange(pop.n_workplaces), m_w)
        sigma = workplace_sigma(pop, seed, step)            # slot base+p -> local index
        posof = np.empty(len(sigma), dtype=np.int64)
        posof[base[owner] + sigma] = np.arange(len(sigma)) - base[owner]
        shifts = work_shifts_all(pop, seed, step, spec.colleague_draws)
        mem = pop.wp_members.astype(np.int64)
        m_i = m_w[owner]
        ok_w = (m_i >= 2) & alive[mem]
        for j in range(spec.colleague_draws):
            r = shifts[owner, j]
            for sign in (1, -1):
                q = np.mod(posof + sign * r, np.maximum(m_i, 1))
                src = mem[base[owner] + sigma[base[owner] + q]]
                ok = ok_w & alive[src]
                S.append(src[ok]); D.append(mem[ok]); K.append(np.ones(int(ok.sum()), np.int8))
    # random slots
    if n >= 2:
        cnt = random_counts(seed, step, n, pop.poisson_table(), dead)
        for j in range(spec.random_slots):
            pi = random_permutation(n, seed, step, j)
            inv = np.empty(n, dtype=np.int64)
            inv[pi] = ids
            ok = (j < cnt) & (pi != ids) & alive & alive[pi]
            S.append(pi[ok]); D.append(ids[ok]); K.append(np.full(int(ok.sum()), 2, np.int8))
            ok = (inv != ids) & (j < cnt[inv]) & alive
            S.append(inv[ok]); D.append(ids[ok]); K.append(np.full(int(ok.sum()), 2, np.int8))
    src = np.concatenate(S).astype(np.int32) if S else np.empty(0, np.int32)
    dst = np.concatenate(D).astype(np.int32) if D else np.empty(0, np.int32)
    kind = np.concatenate(K).astype(np.int8) if K else np.empty(0, np.int8)
    if not canonical:
        return src, dst, kind
    o = np.lexsort((kind, src, dst))
    return src[o], dst[o], kind[o]

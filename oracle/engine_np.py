"""Numpy restatement of the reference step engine — TEST INFRASTRUCTURE.

Restates `pkg/src/epivec/engine.py` (phase order 1-7 of its docstring,
lines 1-17) over any object with the `AgentColumns` attributes.  Delays use
scipy's ppf per draw exactly as `progression.py:48-62, 85-87, 137-162` do, so
this oracle also checks the device's threshold tables independently.

Parameter objects (DiseaseParams, ProgressionTable, InterventionConfig) are
duck-typed: the reference's own classes and the mirror classes in
`paper_2110_04421_b200` both work.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import rng_np

NEVER = -1
S, ASYM, PRE_MILD, PRE_SEV, MILD, SEV, HOSP, ICU, REC, VAC, DEAD = range(11)
INFECTIOUS = np.zeros(11, bool); INFECTIOUS[1:6] = True         # stages.py:63-66
ASYM_LIKE = np.zeros(11, bool); ASYM_LIKE[1:4] = True           # stages.py:68-70
ACTIVE = np.zeros(11, bool); ACTIVE[1:8] = True                 # stages.py:72-77

P_INF, P_INF_EDGE, P_ENTRY, P_BRANCH, P_DELAY = 1, 2, 3, 4, 5      # rng.py:37-57
P_TPOS, P_TTURN, P_QDROP, P_DEN, P_APP, P_VAX = 6, 7, 8, 9, 10, 11


@dataclass
class Events:
    """engine.py:41-52"""
    step: int
    n_edges: int = 0
    new_infections: int = 0
    deaths: int = 0
    hospitalizations: int = 0
    tests_administered: int = 0
    doses_given: int = 0
    notifications_sent: int = 0


def _is_sterilizing(iv) -> bool:
    return int(iv.vaccine.immunity_mode) == 0


def target_mask(cols, sterilizing):
    """engine.py:112-117: susceptible, and not immune under sterilizing mode."""
    m = cols.stage == S
    return m & ~cols.immune if sterilizing else m


def hazard(cols, disease, step, graph, sterilizing):
    """engine.py:77-110.

    Sources are valid while infectious, out of quarantine and 1 <= t <= t_max.
    Valid edges are put in canonical (dst, src, kind) order and the per-edge
    term is evaluated with the pinned factor order
    ((((rate*S[age_d])*A)*B[k])/Ibar)*w[t]; np.bincount then adds the terms of
    each dst sequentially in that order.
    """
    n = cols.n_agents
    out = np.zeros(n, dtype=np.float64)
    if len(graph.src):
        src = np.asarray(graph.src); dst = np.asarray(graph.dst); kind = np.asarray(graph.kind)
        t = step - cols.infected_at[src].astype(np.int64)
        ok = (INFECTIOUS[cols.stage[src]] & (cols.quarantine_until[src] <= step)
              & (t >= 1) & (t <= disease.t_max))
        keep = np.flatnonzero(ok)
        if len(keep):
            s, d, k, tt = src[keep], dst[keep], kind[keep], t[keep]
            o = np.lexsort((k, s, d))
            s, d, k, tt = s[o], d[o], k[o], tt[o]
            a = np.where(ASYM_LIKE[cols.stage[s]], disease.asymptomatic_factor, 1.0)
            term = disease.rate_scale * disease.age_susceptibility[cols.age_band[d]]
            term = term * a
            term = term * disease.network_scale[k]
            term = term / disease.mean_daily_interactions
            term = term * disease.day_weights[tt]
            out = np.bincount(d, weights=term, minlength=n)
    out[~target_mask(cols, sterilizing)] = 0.0
    return out


def edge_terms(cols, disease, step, graph):
    """Valid incident hazards in canonical (dst, src, kind) order, zero terms
    dropped: the contributions of oracle.py:126-144, sorted as oracle.py:178."""
    src = np.asarray(graph.src); dst = np.asarray(graph.dst); kind = np.asarray(graph.kind)
    if not len(src):
        e = np.empty(0, np.int64)
        return e, e, e, np.empty(0)
    t = step - cols.infected_at[src].astype(np.int64)
    ok = (INFECTIOUS[cols.stage[src]] & (cols.quarantine_until[src] <= step)
          & (t >= 1) & (t <= disease.t_max))
    keep = np.flatnonzero(ok)
    s, d, k, tt = src[keep], dst[keep], kind[keep], t[keep]
    o = np.lexsort((k, s, d))
    s, d, k, tt = s[o], d[o], k[o], tt[o]
    a = np.where(ASYM_LIKE[cols.stage[s]], disease.asymptomatic_factor, 1.0)
    term = disease.rate_scale * disease.age_susceptibility[cols.age_band[d]]
    term = term * a
    term = term * disease.network_scale[k]
    term = term / disease.mean_daily_interactions
    term = term * disease.day_weights[tt]
    nz = term != 0.0
    return d[nz].astype(np.int64), s[nz].astype(np.int64), k[nz].astype(np.int64), term[nz]


def pick(rule, age_bands, u):
    """progression.py:117-123: j = #(u >= cum[age]) clipped to the last target."""
    j = (u[:, None] >= rule.cum_probs[age_bands]).sum(axis=1)
    j = np.minimum(j, len(rule.targets) - 1)
    return np.array([int(t) for t in rule.targets], dtype=np.int8)[j]


def schedule(table, stages, age_bands, u_branch, u_delay):
    """progression.py:137-162 (absorbing stages get NEVER/NEVER)."""
    n = len(stages)
    nxt = np.full(n, NEVER, dtype=np.int8)
    delay = np.full(n, NEVER, dtype=np.int64)
    for s, rule in table.rules.items():
        if int(s) == S:
            continue
        idx = np.flatnonzero(stages == int(s))
        if not len(idx):
            continue
        chosen = pick(rule, age_bands[idx], u_branch[idx])
        nxt[idx] = chosen
        for j, spec in enumerate(rule.durations):
            sel = idx[chosen == int(rule.targets[j])]
            if len(sel):
                delay[sel] = np.maximum(np.rint(spec.quantile(u_delay[sel])), 1.0).astype(np.int64)
    return nxt, delay


def priority_order(strategy, elderly_band, age_band, dose2, ids):
    """interventions.py:119-142: lexsort by (group, -age, dose rank, id)."""
    strategy = int(strategy)
    if strategy == 0:
        group = np.where(dose2, 0, 1)
    elif strategy == 1:
        group = np.where(dose2, 1, 0)
    else:
        group = np.where(age_band >= elderly_band, 0, np.where(dose2, 2, 1))
    return np.lexsort((ids, dose2.astype(np.int8), -age_band.astype(np.int64), group))


class ContactRing:
    """interventions.py:145-178: edges of the last `lookback` pushed graphs."""

    def __init__(self, lookback):
        self.lookback = lookback
        self.items = []

    def push(self, graph):
        self.items.append((np.asarray(graph.src), np.asarray(graph.dst)))
        if len(self.items) > self.lookback:
            self.items.pop(0)

    def contacts_of(self, agents):
        if not self.items or not len(agents):
            return np.empty(0, dtype=np.int32)
        top = int(agents.max()) + 1
        flag = np.zeros(top, dtype=bool)
        flag[agents] = True
        found = []
        for src, dst in self.items:
            if not len(src):
                continue
            hit = np.zeros(len(src), dtype=bool)
            low = src < top
            hit[low] = flag[src[low]]
            if hit.any():
                found.append(dst[hit])
        if not found:
            return np.empty(0, dtype=np.int32)
        return np.unique(np.concatenate(found)).astype(np.int32)


class OracleEngine:
    """Restatement of `Engine` (engine.py:55-347) — same constructor shape."""

    def __init__(self, cols, disease, table, interventions, seed, check_invariants=False,
                 infection_mode="aggregate"):
        if infection_mode not in ("aggregate", "independent"):
            raise ValueError(f"unknown infection mode {infection_mode!r}")
        self.infection_mode = infection_mode
        self.cols, self.disease, self.table, self.iv = cols, disease, table, interventions
        self.seed = seed
        self.clock = 0
        self.vaccination_open = False
        self.check = check_invariants
        self.sterilizing = _is_sterilizing(interventions)
        self.ring = ContactRing(interventions.den.lookback) if interventions.den_enabled else None
        self.everyone = np.arange(cols.n_agents, dtype=np.int64)

    def u(self, purpose, ids, k=0):
        return rng_np.uniforms(self.seed, self.clock, purpose, ids, k)

    def gather_exposure(self, graph):
        return hazard(self.cols, self.disease, self.clock, graph, self.sterilizing)

    # engine.py:121-151
    def step(self, graph):
        c, t = self.cols, self.clock
        if graph.step != t:
            raise ValueError(f"graph built for step {graph.step}, engine clock is {t}")
        ev = Events(step=t, n_edges=len(graph.src))
        self._transmit(graph, ev)
        symptomatic = self._progress(ev)
        if self.iv.testing_enabled:
            self._sample_tests(symptomatic, ev)
            self._deliver_tests(ev)
        if self.iv.quarantine_enabled:
            self._dropout()
        if self.iv.vaccination_enabled:
            self._vaccinate(ev)
        if self.ring is not None:
            self.ring.push(graph)
        self.clock += 1
        return ev

    # engine.py:153-175
    def _transmit(self, graph, ev):
        c, t = self.cols, self.clock
        if self.infection_mode == "independent":
            hit = self._independent_hits(graph)
        else:
            lam = self.gather_exposure(graph)
            p = 1.0 - np.exp(-lam)
            hit = np.flatnonzero(target_mask(c, self.sterilizing) & (self.u(P_INF, self.everyone) < p))
        if not len(hit):
            return
        entry = pick(self.table.rules[S], c.age_band[hit], self.u(P_ENTRY, hit))
        if not self.sterilizing:
            entry = np.where(c.immune[hit], np.int8(ASYM), entry)
        c.stage[hit] = entry
        c.infected_at[hit] = t
        nxt, delay = schedule(self.table, entry, c.age_band[hit],
                              self.u(P_BRANCH, hit), self.u(P_DELAY, hit))
        c.next_stage[hit] = nxt
        c.next_transition_at[hit] = t + delay
        ev.new_infections = len(hit)

    # oracle.py:185-192 (independent-edges mode): contribution j of target d
    # infects with its own draw u(seed, t, INFECTION_EDGE, d, k=j) < 1 - exp(-h_j)
    def _independent_hits(self, graph):
        c, t = self.cols, self.clock
        d, _, _, term = edge_terms(c, self.disease, t, graph)
        if not len(d):
            return np.empty(0, dtype=np.int64)
        first = np.searchsorted(d, d, side="left")
        j = np.arange(len(d)) - first
        u = rng_np.uniforms(self.seed, t, P_INF_EDGE, d, np.asarray(j, dtype=np.uint64))
        hit = np.unique(d[u < 1.0 - np.exp(-term)])
        return hit[target_mask(c, self.sterilizing)[hit]]

    # engine.py:177-200
    def _progress(self, ev):
        c, t = self.cols, self.clock
        due = np.flatnonzero(c.next_transition_at == t)
        if not len(due):
            return np.empty(0, dtype=np.int64)
        dest = c.next_stage[due].copy()
        c.stage[due] = dest
        ev.deaths = int((dest == DEAD).sum())
        ev.hospitalizations = int((dest == HOSP).sum())
        symptomatic = due[(dest == MILD) | (dest == SEV)]
        final = (dest == REC) | (dest == DEAD)
        c.next_stage[due[final]] = NEVER
        c.next_transition_at[due[final]] = NEVER
        rest = due[~final]
        if len(rest):
            nxt, delay = schedule(self.table, c.stage[rest], c.age_band[rest],
                                  self.u(P_BRANCH, rest), self.u(P_DELAY, rest))
            c.next_stage[rest] = nxt
            c.next_transition_at[rest] = t + delay
        return symptomatic

    # engine.py:202-227
    def _sample_tests(self, symptomatic, ev):
        c, t = self.cols, self.clock
        den_due = np.flatnonzero(c.den_test_due_at == t)
        c.den_test_due_at[den_due] = NEVER
        cand = np.unique(np.concatenate([symptomatic, den_due]))
        if not len(cand):
            return
        ids = cand[(c.test_result_at[cand] == NEVER) & (c.stage[cand] != DEAD)]
        if not len(ids):
            return
        kind = self.iv.test_kind
        up = self.u(P_TPOS, ids)
        pos = np.where(ACTIVE[c.stage[ids]], up < kind.detection_prob,
                       up < self.iv.false_positive_prob)
        span = kind.turnaround_max - kind.turnaround_min + 1
        turn = kind.turnaround_min + (self.u(P_TTURN, ids) * span).astype(np.int64)
        c.test_sample_at[ids] = t
        c.test_result_at[ids] = t + turn
        c.test_positive[ids] = pos
        ev.tests_administered = len(ids)

    # engine.py:229-262
    def _deliver_tests(self, ev):
        c, t = self.cols, self.clock
        due = np.flatnonzero(c.test_result_at == t)
        if not len(due):
            return
        pos = due[c.test_positive[due]]
        c.test_result_at[due] = NEVER
        c.test_positive[due] = False
        if self.iv.quarantine_enabled and len(pos):
            c.quarantine_until[pos] = t + self.iv.quarantine_duration
            c.quarantine_started_at[pos] = t
        if self.iv.den_enabled and len(pos):
            notifiers = pos[c.has_den_app[pos]]
            if not len(notifiers) or self.ring is None:
                return
            contacts = self.ring.contacts_of(notifiers)
            if not len(contacts):
                return
            ok = (c.has_den_app[contacts] & (c.quarantine_until[contacts] <= t)
                  & (c.stage[contacts] != DEAD))
            told = contacts[ok]
            if not len(told):
                return
            ev.notifications_sent = len(told)
            comply = told[self.u(P_DEN, told) < self.iv.den.compliance_prob]
            c.den_test_due_at[comply] = t + 1

    # engine.py:264-273
    def _dropout(self):
        c, t = self.cols, self.clock
        q = np.flatnonzero((c.quarantine_until > t) & (c.quarantine_started_at < t))
        if len(q):
            leave = q[self.u(P_QDROP, q) < self.iv.quarantine_dropout]
            c.quarantine_until[leave] = t

    # engine.py:275-347
    def _vaccinate(self, ev):
        c, t, pol = self.cols, self.clock, self.iv.vaccine
        due = np.flatnonzero(c.immunity_check_at == t)
        for dose in (1, 2):
            ids = due[c.immunity_check_dose[due] == dose]
            if len(ids):
                self._immunity(ids, dose)
        if not self.vaccination_open:
            if int(ACTIVE[c.stage].sum()) >= pol.start_trigger * c.n_agents:
                self.vaccination_open = True
        if not self.vaccination_open:
            return
        budget = int(np.rint(pol.daily_rate * c.n_agents))
        if budget <= 0:
            return
        blocked = (c.stage == DEAD) | (c.stage == HOSP) | (c.stage == ICU)
        d1 = (c.vaccine_status == 0) & ~blocked
        d2 = ((c.vaccine_status == 1) & (c.dose1_at != NEVER)
              & (t >= c.dose1_at + pol.dose_gap) & ~blocked)
        elig = np.flatnonzero(d1 | d2)
        if not len(elig):
            return
        order = priority_order(pol.strategy, pol.elderly_band, c.age_band[elig], d2[elig], elig)
        take = elig[order][:budget]
        ev.doses_given = len(take)
        second = d2[take]
        first, sec = take[~second], take[second]
        if len(first):
            c.vaccine_status[first] = 1
            c.dose1_at[first] = t
            c.immunity_check_at[first] = t + pol.dose1_latency
            c.immunity_check_prob[first] = pol.dose1_efficacy
            c.immunity_check_dose[first] = 1
            if pol.dose1_latency == 0:
                self._immunity(first, 1)
        if len(sec):
            c.vaccine_status[sec] = 2
            c.dose2_at[sec] = t
            e1, e2 = pol.dose1_efficacy, pol.dose2_efficacy
            topup = 0.0 if e1 >= 1.0 else max(0.0, (e2 - e1) / (1.0 - e1))
            prob = np.where(c.immunity_check_at[sec] != NEVER, pol.dose2_efficacy, topup)
            prob = np.where(c.immune[sec], 0.0, prob)
            c.immunity_check_at[sec] = t + pol.dose2_latency
            c.immunity_check_prob[sec] = prob
            c.immunity_check_dose[sec] = 2
            if pol.dose2_latency == 0:
                self._immunity(sec, 2)

    def _immunity(self, ids, dose):
        c = self.cols
        ok = ids[(self.u(P_VAX, ids, dose) < c.immunity_check_prob[ids]) & (c.stage[ids] == S)]
        c.immune[ok] = True
        if self.sterilizing:
            c.stage[ok] = VAC
        c.immunity_check_at[ids] = NEVER
        c.immunity_check_prob[ids] = 0.0
        c.immunity_check_dose[ids] = 0


SERIES_COLUMNS = (["step"] + [f"n_{n}" for n in (
    "susceptible", "asymptomatic", "presymptomatic_mild", "presymptomatic_severe",
    "mild_symptomatic", "severe_symptomatic", "hospitalized", "critical_icu",
    "recovered", "vaccinated", "dead")] + [
    "cumulative_infections", "cumulative_deaths", "in_hospital_or_icu",
    "new_infections", "tests_administered", "doses_given", "notifications_sent"])


def series_row(cols, ev):
    """runner.py:101-116 — one 19-column time-series row."""
    counts = np.bincount(cols.stage, minlength=11)
    return np.array([ev.step, *counts, int((cols.infected_at != NEVER).sum()),
                     counts[DEAD], counts[HOSP] + counts[ICU], ev.new_infections,
                     ev.tests_administered, ev.doses_given, ev.notifications_sent],
                    dtype=np.int64)

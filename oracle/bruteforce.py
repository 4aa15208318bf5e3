"""Brute-force references for toy inputs -- TEST INFRASTRUCTURE ONLY.

Pure-Python, float64, written from PAPER.md without the fixed-point encoding:
  literal_decide   Algorithm 1 with the real-valued Eq. 3-4
                   (P:300-318), Eq. 5, Eq. 6 and the
                   queue prediction of P:347-353; Eq. 7 argmin.
  mini_replay      an independent executor of a given action sequence under
                   exclusive time-division execution.
  tree_min_violations
                   exhaustive search over every (m, e, b) action sequence of
                   a toy trace (the "global optimum" the paper calls
                   impractical) -- a bound the greedy must respect.
"""
from __future__ import annotations

import math


def urgency(w, tau, C):
    """Eq. 3: f(w) = min(exp(w/tau - 1), C)."""
    return min(math.exp(w / tau - 1.0), float(C))


def stability_score(pred_waits, tau, C):
    """Eq. 4: S = sum over queues and tasks of f(w)."""
    return sum(urgency(w, tau, C) for q in pred_waits for w in q)


def batch_size(qlen, b_max, bs):
    """Eq. 5, B* = min(|Q|, B_max), snapped to the largest profiled size (Q8)."""
    cap = min(qlen, b_max)
    return max(b for b in bs if b <= cap)


def exit_point(lat_row_at_b, allowed, w_max, tau):
    """Eq. 6 by linear search; (deepest feasible, True) else (shallowest allowed, False)."""
    best = None
    for e, L in enumerate(lat_row_at_b):
        if allowed[e] and w_max + L <= tau:
            best = e
    if best is None:
        return min(e for e in range(len(allowed)) if allowed[e]), False
    return best, True


def predict(waits, m, B, L):
    """Queue status prediction: drop the B served tasks of Q_m,
    add L to every remaining wait, no future arrivals."""
    out = []
    for m2, q in enumerate(waits):
        rest = q[B:] if m2 == m else q
        out.append([w + L for w in rest])
    return out


def literal_decide(prof, tau, C, b_max, waits):
    """waits[m] = head-first list of current waits.  Returns (m*, e*, B*, scores
    dict m -> (S, e, B, feasible)) or None when every queue is empty."""
    bs = [int(b) for b in prof.bs]
    scores = {}
    for m, q in enumerate(waits):
        if not q:
            continue
        B = batch_size(len(q), b_max, bs)
        bi = bs.index(B)
        row = [int(prof.lat[m, e, bi]) for e in range(prof.E)]
        e, feas = exit_point(row, [bool(x) for x in prof.mask[m]], q[0], tau)
        L = row[e]
        S = stability_score(predict(waits, m, B, L), tau, C)
        scores[m] = (S, e, B, feas, L)
    if not scores:
        return None
    m_star = min(scores, key=lambda m: (scores[m][0], m))
    return m_star, scores[m_star][1], scores[m_star][2], scores


def mini_replay(arrivals, actions, lat_of):
    """Execute a fixed action list [(m, e, B)] under time-division execution.

    Each action starts when the GPU is free and its B oldest pending requests
    of queue m have arrived (work-conserving: start = max(free, arrival of the
    B-th request ... but never before the previous completion)).  Returns the
    per-model completion lists.  lat_of(m, e, B) -> us.
    """
    M = len(arrivals)
    head = [0] * M
    comp = [[None] * len(a) for a in arrivals]
    free = min((a[0] for a in arrivals if a), default=0)
    for (m, e, B) in actions:
        start = max(free, arrivals[m][head[m] + B - 1])
        done = start + lat_of(m, e, B)
        for i in range(head[m], head[m] + B):
            comp[m][i] = done
        head[m] += B
        free = done
    return comp


def _tree(arrivals, t, head, prof, tau, b_max, bs, acc_viol, best, W_counter):
    M = len(arrivals)
    tail = [sum(1 for x in arrivals[m] if x <= t) for m in range(M)]
    remaining = sum(len(arrivals[m]) - head[m] for m in range(M))
    if remaining == 0:
        best[0] = min(best[0], acc_viol)
        return
    if all(tail[m] == head[m] for m in range(M)):
        nt = min(arrivals[m][tail[m]] for m in range(M) if tail[m] < len(arrivals[m]))
        _tree(arrivals, nt, head, prof, tau, b_max, bs, acc_viol, best, W_counter)
        return
    if acc_viol >= best[0]:
        return
    for m in range(M):
        n = tail[m] - head[m]
        if n == 0:
            continue
        for bi, B in enumerate(bs):
            if B > min(n, b_max):
                continue
            for e in range(prof.E):
                if not prof.mask[m][e]:
                    continue
                L = int(prof.lat[m, e, bi])
                done = t + L
                v = sum(1 for i in range(head[m], head[m] + B) if done - arrivals[m][i] > tau)
                head[m] += B
                _tree(arrivals, done, head, prof, tau, b_max, bs, acc_viol + v, best, W_counter)
                head[m] -= B


def tree_min_violations(arrivals, prof, tau, b_max):
    """Minimum achievable violation count (warmup 0) over every action sequence
    of a non-idling scheduler on a toy trace (exponential; M<=3, <=8 requests)."""
    bs = [int(b) for b in prof.bs]
    t0 = min(a[0] for a in arrivals if a)
    best = [math.inf]
    _tree([list(map(int, a)) for a in arrivals], t0, [0] * len(arrivals), prof, tau, b_max, bs, 0,
          best, None)
    return best[0]


# the paper's baselines (§VI-A) and ablations (§VI-H),
# read as DESIGN.md Q26; names as in SPEC's policy_decide
POLICY_IDS = {"edgeserving": 0, "all_final": 1, "all_early": 2, "ee_lqf": 3, "ee_edf": 4, "allfinal_da": 5,
              "ours_bs1": 6, "symphony": 7, "grid": 8}


def literal_policy_decide(prof, tau, C, b_max, waits, policy):
    """One decision of `policy` on head-first waits, float64 scores.  Returns
    (m*, e*, B*, feasible, scores) with scores = {m: S} for the scoring
    policies ({} otherwise), or None when every queue is empty."""
    bs = [int(b) for b in prof.bs]
    nonempty = [m for m, q in enumerate(waits) if q]
    if not nonempty:
        return None

    def params(m):
        q = waits[m]
        B = 1 if policy == "ours_bs1" else batch_size(len(q), b_max, bs)  # "fixes batch size to 1"
        bi = bs.index(B)
        row = [int(prof.lat[m, e, bi]) for e in range(prof.E)]
        allowed = [bool(x) for x in prof.mask[m]]
        if policy in ("all_final", "allfinal_da"):  # "always executes them at the deepest exit"
            e = max(i for i in range(prof.E) if allowed[i])
            feas = q[0] + row[e] <= tau
        elif policy == "all_early":  # "always executes them at the shallowest exit"
            e = min(i for i in range(prof.E) if allowed[i])
            feas = q[0] + row[e] <= tau
        else:  # profile-based exit selection, Eq. 6
            e, feas = exit_point(row, allowed, q[0], tau)
        return e, B, feas, row[e]

    if policy in ("all_final", "all_early", "ee_lqf"):  # longest queue first
        m_star = min(nonempty, key=lambda m: (-len(waits[m]), m))
        e, B, feas, _ = params(m_star)
        return m_star, e, B, feas, {}
    if policy == "ee_edf":  # least remaining SLO slack tau - w of the oldest task
        m_star = min(nonempty, key=lambda m: (tau - waits[m][0], m))
        e, B, feas, _ = params(m_star)
        return m_star, e, B, feas, {}
    scores = {}
    for m in nonempty:
        e, B, feas, L = params(m)
        scores[m] = stability_score(predict(waits, m, B, L), tau, C)
    m_star = min(scores, key=lambda m: (scores[m], m))
    e, B, feas, _ = params(m_star)
    return m_star, e, B, feas, scores


def symphony_replay_us(prof, tau, b_max, arrivals):
    """Deferred batching (Symphony; Q27) simulated one
    microsecond at a time -- no event jumps: whenever the GPU is free at
    instant t, admit arrivals <= t; a queue is triggered when its head wait +
    L(m, deepest allowed exit, B*) >= tau or it holds >= B_max tasks; the
    triggered queue with the largest head wait + L is served (ties lowest m),
    the batch runs exclusively for L; with none triggered the GPU stays idle
    for one microsecond.  arrivals[m] = sorted list.  Returns the dispatch
    list [(t, m, e, B)] and the completion time of every request."""
    bs = [int(b) for b in prof.bs]
    M = len(arrivals)
    head = [0] * M
    tail = [0] * M
    done = [[None] * len(a) for a in arrivals]
    total = sum(len(a) for a in arrivals)
    served = 0
    t = min(a[0] for a in arrivals if a)
    out = []
    while served < total:
        for m in range(M):
            while tail[m] < len(arrivals[m]) and arrivals[m][tail[m]] <= t:
                tail[m] += 1
        best, best_need = None, -1
        for m in range(M):
            n = tail[m] - head[m]
            if n == 0:
                continue
            B = batch_size(n, b_max, bs)
            e = max(i for i in range(prof.E) if prof.mask[m][i])
            L = int(prof.lat[m, e, bs.index(B)])
            need = t - arrivals[m][head[m]] + L
            if (need >= tau or n >= b_max) and need > best_need:
                best, best_need = m, need
        if best is None:
            t += 1
            continue
        m = best
        n = tail[m] - head[m]
        B = batch_size(n, b_max, bs)
        e = max(i for i in range(prof.E) if prof.mask[m][i])
        L = int(prof.lat[m, e, bs.index(B)])
        out.append((t, m, e, B))
        for i in range(head[m], head[m] + B):
            done[m][i] = t + L
        head[m] += B
        served += B
        t += L
    return out, done


def literal_grid_decide(prof, tau, C, b_max, waits):
    """GRID (f2): every admissible (m, e, b) -- allowed exit, profiled b <=
    min(|Q_m|, B_max) -- scored by the literal float64 Eq. 3-4 on the
    prediction of serving b tasks of Q_m at exit e; argmin of (S, m, e, b).
    Returns (m, e, b, feasible, {(m, e, b): S}) or None."""
    bs = [int(b) for b in prof.bs]
    scores = {}
    for m, q in enumerate(waits):
        if not q:
            continue
        for e in range(prof.E):
            if not prof.mask[m][e]:
                continue
            for bi, b in enumerate(bs):
                if b > min(len(q), b_max):
                    break
                L = int(prof.lat[m, e, bi])
                scores[(m, e, b)] = stability_score(predict(waits, m, b, L), tau, C)
    if not scores:
        return None
    m, e, b = min(scores, key=lambda k: (scores[k], k))
    L = int(prof.lat[m, e, bs.index(b)])
    return m, e, b, waits[m][0] + L <= tau, scores

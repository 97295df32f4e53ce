"""Restatement of the reference's discrete-epoch replay (collsched
simulator.py:58-235). TEST INFRASTRUCTURE ONLY: used by tests/ to check
schedules this package emits, never by the product path.

Copy-capable / no-copy switch modes; the hyper-edge mode (legacy switch
rewrite) is not needed for LP schedules and is omitted.
"""

from __future__ import annotations

from fractions import Fraction

WHOLE = 1.0 - 1e-9


def _snap(x):
    if isinstance(x, Fraction):
        return x
    if isinstance(x, int):
        return Fraction(x)
    return Fraction(x).limit_denominator(10 ** 12)


def _ceil(q):
    return -int((-q) // 1) if q > 0 else 0


def simulate(events, tau, chunk_size, t, entries, switch_mode="copy", tol=1e-6):
    """events: iterable of (source, chunk, src, dst, epoch, fraction).
    Returns dict(violations=[(kind, location, epoch)], completion_epoch,
    per_entry=dict)."""
    tau_q = _snap(tau)
    chunk = Fraction(chunk_size)
    caps = {(e.src, e.dst): _snap(e.capacity) * tau_q / chunk for e in t.edges}   # simulator.py:80-82
    events = [tuple(e) for e in events]
    whole_only = all(e[5] >= WHOLE for e in events)
    kap = {pair: (max(1, _ceil(1 / c)) if whole_only else 1) for pair, c in caps.items()}
    widen = max(kap.values(), default=1) - 1
    delta = {(e.src, e.dst): _ceil(_snap(e.alpha) / tau_q) + widen for e in t.edges}
    events.sort(key=lambda e: (e[4], str(e[0]), str(e[2]), str(e[3]), e[1]))      # simulator.py:94-95
    viol = []
    copy_from, frac_pool, sw_arr, deliveries = {}, {}, {}, {}
    for s, c, _ in entries:
        copy_from[(s, c, s)] = 0
    entry_index = set(entries)

    def register(s, c, node, arr, qty):                                           # :119-131
        if t.is_switch(node):
            sw_arr.setdefault((s, c, node), []).append(
                {"usable": arr + 1, "qty": qty, "used": 0.0, "whole": qty >= WHOLE})
        elif qty >= WHOLE:
            prev = copy_from.get((s, c, node))
            if prev is None or arr + 1 < prev:
                copy_from[(s, c, node)] = arr + 1
        else:
            frac_pool.setdefault((s, c, node), []).append([arr + 1, qty])
        if (s, c, node) in entry_index:
            deliveries.setdefault((s, c, node), []).append((arr, qty))

    def draw(s, c, node, k, qty):                                                 # :133-163
        if t.is_switch(node):
            recs = [r for r in sw_arr.get((s, c, node), ()) if r["usable"] == k]
            if switch_mode != "no-copy":
                for r in recs:
                    if r["whole"]:
                        r["used"] += qty
                        return True
            rem = qty
            for r in recs:
                free = r["qty"] - r["used"]
                if free > tol:
                    take = min(free, rem)
                    r["used"] += take
                    rem -= take
                    if rem <= tol:
                        return True
            return rem <= tol
        ready = copy_from.get((s, c, node))
        if ready is not None and ready <= k:
            return True
        rem = qty
        for rec in frac_pool.get((s, c, node), ()):
            if rec[0] <= k and rec[1] > tol:
                take = min(rec[1], rem)
                rec[1] -= take
                rem -= take
                if rem <= tol:
                    return True
        return rem <= tol

    for s, c, i, j, k, f in events:                                               # :165-170
        if not draw(s, c, i, k, f):
            viol.append(("causality", f"{i!r} lacks chunk {c} of {s!r}", k))
        register(s, c, j, k + delta[(i, j)], f)
    load, max_epoch = {}, -1                                                      # :211-223
    for s, c, i, j, k, f in events:
        load[(i, j, k)] = load.get((i, j, k), 0.0) + f
        max_epoch = max(max_epoch, k)
    for (i, j), cap in caps.items():
        w = kap[(i, j)]
        budget = float(w * cap)
        for k in range(max_epoch + 1):
            total = sum(load.get((i, j, k2), 0.0) for k2 in range(k - w + 1, k + 1))
            if total > budget * (1 + tol) + tol:
                viol.append(("capacity", f"({i!r},{j!r})", k))
    for (s, c, sw), recs in sorted(sw_arr.items(), key=str):                      # :226-235
        for r in recs:
            if switch_mode == "no-copy" or not r["whole"]:
                if r["qty"] - r["used"] > tol:
                    viol.append(("switch-buffer", f"chunk {c} of {s!r} rests at {sw!r}", r["usable"]))
            elif r["used"] == 0.0:
                viol.append(("switch-buffer", f"chunk {c} of {s!r} rests at {sw!r}", r["usable"]))
    per_entry = {}
    for key in sorted(entry_index, key=str):                                      # :176-189
        acc, done = 0.0, None
        for arr, qty in sorted(deliveries.get(key, ())):
            acc += qty
            if acc >= 1.0 - tol:
                done = arr
                break
        if done is None:
            viol.append(("unmet-demand", f"chunk {key[1]} of {key[0]!r} at {key[2]!r}", -1))
        else:
            per_entry[key] = done
    return {"violations": viol, "completion_epoch": max(per_entry.values(), default=-1),
            "per_entry": per_entry}

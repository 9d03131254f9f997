"""Double-Ring KV rotation schedule (inner ring of size w x outer ring of d_cp/w).

Consumption order per CP rank follows ref ``ring.py:41-61``: CP rank j sits at
position ``p = j mod w`` of inner ring ``r = j // w``; at outer step o, inner
step t it consumes the KV chunk that originated at CP rank

    src(j, o, t) = ((r - o) mod n) * w + (p - t) mod w,      n = d_cp / w.

The B200 runtime additionally needs to know, for each step, *who to send the
chunk it holds to* and *who it receives the next chunk from*. Because every
rank's source sequence is the same permutation shape, the hand-offs form two
fixed patterns (Alg. 2):

* inner step (t -> t+1 within an outer step): send to (r, p+1), recv from
  (r, p-1) — the classic ring inside one inner group;
* outer step (o -> o+1): the chunk a rank consumes first at outer step o+1 is
  ((r-o-1) mod n)*w + p, which at outer step o was consumed first (t=0) by rank
  (r-1, p).  So the outer hop moves the *inner-ring-initial* chunk from ring
  r-1 to ring r, position-preserving.  This is what lets the outer transfer
  start at the beginning of the outer step and overlap all w inner micro-steps.

The backward needs the same walk for the KV chunk plus a travelling dK/dV
accumulator that returns to the chunk's owner at the end (ref has no
distributed backward; this routing is ours and is proven against
the global oracle in tests).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class RingStep:
    outer: int
    inner: int
    source: int  # CP rank whose original KV chunk is consumed at this step


@dataclass(frozen=True)
class RingSchedule:
    d_cp: int
    inner_ring: int
    steps: tuple[tuple[RingStep, ...], ...]  # [cp_rank][step]

    @property
    def outer_rings(self) -> int:
        return self.d_cp // self.inner_ring


def _src(j: int, o: int, t: int, w: int, n: int) -> int:
    ring, pos = divmod(j, w)
    return ((ring - o) % n) * w + (pos - t) % w


def build_ring_schedule(d_cp: int, w: int) -> RingSchedule:
    """Per-CP-rank KV consumption order (ref ``ring.py:41-61``)."""
    if w < 1 or d_cp % w != 0:
        raise ValueError(f"inner ring size {w} must divide d_cp={d_cp}")
    n = d_cp // w
    table = tuple(
        tuple(RingStep(o, t, _src(j, o, t, w, n))
              for o in range(n) for t in range(w))
        for j in range(d_cp))
    return RingSchedule(d_cp, w, table)


@dataclass(frozen=True)
class Transfer:
    """One point-to-point hop a CP rank performs between two steps."""

    kind: str        # "inner" | "outer" | "home"
    send_to: int     # CP rank index receiving our buffer
    recv_from: int   # CP rank index whose buffer we receive


def inner_peers(j: int, w: int) -> tuple[int, int]:
    """(send_to, recv_from) for an inner-ring hop of CP rank j."""
    ring, pos = divmod(j, w)
    return ring * w + (pos + 1) % w, ring * w + (pos - 1) % w


def outer_peers(j: int, d_cp: int, w: int) -> tuple[int, int]:
    """(send_to, recv_from) for an outer-ring hop: same position, ring +-1."""
    n = d_cp // w
    ring, pos = divmod(j, w)
    return ((ring + 1) % n) * w + pos, ((ring - 1) % n) * w + pos


def step_transfers(j: int, d_cp: int, w: int) -> list[Transfer | None]:
    """Hop needed *before* each step s>0 for CP rank j (index 0 is None).

    Before step (o, t>0): inner hop of the chunk consumed at (o, t-1).
    Before step (o>0, 0): outer hop of the chunk consumed at (o-1, 0).
    """
    n = d_cp // w
    out: list[Transfer | None] = [None]
    for o in range(n):
        for t in range(w):
            if o == 0 and t == 0:
                continue
            if t > 0:
                s, r = inner_peers(j, w)
                out.append(Transfer("inner", s, r))
            else:
                s, r = outer_peers(j, d_cp, w)
                out.append(Transfer("outer", s, r))
    return out


def home_transfer(j: int, schedule: RingSchedule) -> Transfer:
    """Final hop of the backward dK/dV accumulator back to its owner.

    Rank j's last consumed chunk is ``last = steps[j][-1].source``; its
    accumulator goes home to CP rank ``last``; rank j receives the accumulator
    of its own chunk from the rank whose last source is j.
    """
    last = schedule.steps[j][-1].source
    sender = next(i for i in range(schedule.d_cp)
                  if schedule.steps[i][-1].source == j)
    return Transfer("home", last, sender)


@dataclass(frozen=True)
class RingPeers:
    """CP-rank indices one rank talks to (all hops are fixed permutations)."""

    inner_to: int
    inner_from: int
    outer_to: int
    outer_from: int
    diag_to: int     # dK/dV accumulator hop across outer steps and the home hop
    diag_from: int


def ring_peers(j: int, d_cp: int, w: int) -> RingPeers:
    n = d_cp // w
    ring, pos = divmod(j, w)

    def idx(r, p):
        return (r % n) * w + (p % w)

    return RingPeers(idx(ring, pos + 1), idx(ring, pos - 1), idx(ring + 1, pos), idx(ring - 1, pos),
                     idx(ring + 1, pos + 1), idx(ring - 1, pos - 1))


def dkv_hop(step: int, d_cp: int, w: int) -> str:
    """Hop of the backward dK/dV accumulator after step `step`: 'inner' while
    the next step stays in the same outer step, else 'diag' (incl. home)."""
    if step == d_cp - 1 or (step + 1) % w == 0:
        return "diag"
    return "inner"


def check_dkv_route(schedule: RingSchedule) -> None:
    """Prove the backward accumulator routing: the accumulator a rank forwards
    after step s reaches exactly the rank that consumes the same chunk at step
    s+1, and after the last step every accumulator lands at its owner."""
    d_cp, w = schedule.d_cp, schedule.inner_ring
    holder = {j: schedule.steps[j][0].source for j in range(d_cp)}  # rank -> chunk of its accumulator
    seen = {c: [] for c in range(d_cp)}
    for j in range(d_cp):
        seen[holder[j]].append(j)
    for s in range(d_cp):
        kind = dkv_hop(s, d_cp, w)
        nxt = {}
        for j in range(d_cp):
            p = ring_peers(j, d_cp, w)
            to = p.inner_to if kind == "inner" else p.diag_to
            nxt[to] = holder[j]
        holder = nxt
        if s + 1 < d_cp:
            for j in range(d_cp):
                want = schedule.steps[j][s + 1].source
                if holder[j] != want:
                    raise AssertionError(f"step {s + 1}: rank {j} holds dKV of {holder[j]}, consumes {want}")
                seen[want].append(j)
    if any(holder[j] != j for j in range(d_cp)):
        raise AssertionError(f"home hop misroutes: {holder}")
    for c, ranks in seen.items():
        if sorted(ranks) != list(range(d_cp)):
            raise AssertionError(f"chunk {c} accumulator visited {ranks}")


def check_walk(schedule: RingSchedule) -> None:
    """Assert the hop patterns reproduce the consumption table exactly.

    Simulates chunk ownership through inner/outer hops and checks each rank
    holds ``steps[j][s].source`` at step s, and that the home hop returns every
    chunk to its owner.
    """
    d_cp, w = schedule.d_cp, schedule.inner_ring
    n = d_cp // w
    cur = [j for j in range(d_cp)]          # chunk held for compute
    first = list(cur)                        # inner-ring-initial chunk this outer step
    for s in range(d_cp):
        o, t = divmod(s, w)
        if s > 0:
            if t > 0:
                nxt = [None] * d_cp
                for j in range(d_cp):
                    to, _ = inner_peers(j, w)
                    nxt[to] = cur[j]
                cur = nxt
            else:
                nxt = [None] * d_cp
                for j in range(d_cp):
                    to, _ = outer_peers(j, d_cp, w)
                    nxt[to] = first[j]
                cur = nxt
                first = list(cur)
        for j in range(d_cp):
            if cur[j] != schedule.steps[j][s].source:
                raise AssertionError(f"rank {j} step {s}: holds {cur[j]}, "
                                     f"schedule says {schedule.steps[j][s].source}")
    home = [None] * d_cp
    for j in range(d_cp):
        home[home_transfer(j, schedule).send_to] = cur[j]
    if home != list(range(d_cp)):
        raise AssertionError(f"home hop misroutes: {home}")
    del n

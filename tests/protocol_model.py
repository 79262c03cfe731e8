"""Exhaustive interleaving explorer for the device engine's round protocol.

TEST INFRASTRUCTURE (the analogue of the reference's verify.py:329-481
explore_interleavings, which runs its engine under every message-delivery
order).  compute-sanitizer is unavailable on this pool, and the engine's races
are between *protocols* -- a controller thread per rank, worker CTAs, peers'
control words over NVLink, and a host reader's pin handshake -- so this models
the controller of csrc/ec_kernels.cu (engine_controller) at the granularity of
its loop sections and explores every interleaving of:

* each rank's controller sections: A (mirror + acknowledge the host pin),
  B (take one request), C (snapshot decision, with the slot-reuse pin check),
  D (issue the round command), E (host publication of a completed round),
  F (round completion: every owner's done word in);
* each owner's workers finishing an issued round (its done word);
* the host: back-to-back offers (the pipelined pattern that lets round g+1 be
  snapshotted and issued while round g is in flight, EcDesc::lead = 2) and a
  reader that pins the latest published generation with ec_wait's handshake
  (pin, wait for the acknowledgement, re-check done_gen1) and reads its slot.

Checked in every reachable state: a pinned slot is never written (no round
X != G with X = G mod R is issued while a reader reads G), rounds publish in
order, at most `lead` rounds are in flight, all ranks agree on every
generation's mask; in every terminal state every round completed everywhere.

`ack_publishes=False` models the controller before the fix that publishes
completed rounds to the host before acknowledging a pin: the explorer finds
the slot-reuse race that fix closes.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

INF = 1 << 30


@dataclass(frozen=True)
class Rank:
    pc: str = "A"            # next controller section
    g: int = 0               # oldest unpublished generation
    n_iss: int = 0           # rounds in flight (g .. g + n_iss - 1)
    snapped: bool = False    # open generation go = g + n_iss snapshotted
    contrib: bool = False    # this rank's offer for go accepted
    contributed: int = -1
    queue: tuple = ()        # posted, unprocessed offers (round numbers)
    pub: int = -1            # completed round awaiting host publication (-1: none)
    host_done: int = 0       # host-visible done_gen1
    pin_mirror: int = INF    # the controller's copy of the host pin
    acked: int = 0           # pin sequence acknowledged
    # host side
    next_offer: int = 0
    pin: int = INF           # host pin word
    pin_seq: int = 0
    reader: tuple = ("idle",)   # ("idle",) | ("ack", G, seq) | ("read", G) | ("done",)


@dataclass(frozen=True)
class State:
    ranks: tuple
    snap: tuple              # snap_from[q] = last generation q snapshotted + 1
    done: tuple              # done_from[q] = last generation q's workers finished + 1
    issued: tuple            # per owner q: rounds issued by q, not yet done (generations)
    hi: tuple = ()           # per owner q: highest generation q ever issued (-1: none)


@dataclass
class Report:
    states: int = 0
    terminals: int = 0
    violations: list = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not self.violations and self.terminals > 0


def explore(p: int = 2, rounds: int = 3, R: int = 3, lead: int = 2, reader_rank: int = 0,
            ack_publishes: bool = True, preposted: bool = False, reader_lead: int | None = None,
            max_states: int = 2_000_000) -> Report:
    """preposted=True: every offer is queued before the first controller step
    (the burst rounds_pipelined issues); False interleaves the posts too.
    reader_lead: the lead the host reader's re-check assumes (default: the
    engine's); a reader assuming 1 against an engine at 2 is the wrong margin."""
    rl = lead if reader_lead is None else reader_lead
    r0 = Rank(queue=tuple(range(rounds)), next_offer=rounds) if preposted else Rank()
    init = State(ranks=tuple(r0 for _ in range(p)), snap=(0,) * p, done=(0,) * p,
                 issued=((),) * p, hi=(-1,) * p)
    rep = Report()
    seen = set()
    stack = [init]

    def set_rank(s: State, r: int, **kw) -> State:
        rs = list(s.ranks)
        rs[r] = replace(rs[r], **kw)
        return replace(s, ranks=tuple(rs))

    def publish(s: State, r: int) -> State:
        rk = s.ranks[r]
        if rk.pub < 0:
            return s
        return set_rank(s, r, host_done=rk.pub + 1, pub=-1)

    def successors(s: State, only_ctrl_of=None):
        """Every next state; with only_ctrl_of=r, just rank r's controller step."""
        out = []
        for r in range(p):
            if only_ctrl_of is not None and r != only_ctrl_of:
                continue
            rk = s.ranks[r]
            go = rk.g + rk.n_iss
            open_ok = rk.n_iss < lead
            nxt = {"A": "B", "B": "C", "C": "D", "D": "E", "E": "F", "F": "A"}[rk.pc]
            if rk.pc == "A":
                t = s
                if rk.pin != rk.pin_mirror or rk.acked != rk.pin_seq:
                    if ack_publishes:
                        t = publish(t, r)
                    t = set_rank(t, r, pin_mirror=rk.pin, acked=rk.pin_seq)
                out.append(set_rank(t, r, pc=nxt))
            elif rk.pc == "B":
                t = s
                if open_ok and rk.queue:
                    off = rk.queue[0]
                    allowed = rk.n_iss == 0 or off == go
                    deferred = off == go + 1 and (rk.snapped or rk.contributed == go)
                    if allowed and not deferred:
                        q = rk.queue[1:]
                        if off == go and not rk.snapped:      # accepted (all-arrive solo)
                            t = set_rank(t, r, queue=q, contrib=True, contributed=off)
                        else:                                  # refused (late)
                            t = set_rank(t, r, queue=q)
                out.append(set_rank(t, r, pc=nxt))
            elif rk.pc == "C":
                t = s
                if (open_ok and not rk.snapped and rk.contrib and go < rounds
                        and (rk.n_iss == 0 or rk.contributed == go)):
                    ok = not (go >= R and rk.pin_mirror <= go - R)
                    if ok:
                        snap = list(s.snap)
                        snap[r] = go + 1
                        t = replace(set_rank(t, r, snapped=True), snap=tuple(snap))
                out.append(set_rank(t, r, pc=nxt))
            elif rk.pc == "D":
                if open_ok and rk.snapped and all(x >= go + 1 for x in s.snap):
                    iss = list(s.issued)
                    iss[r] = iss[r] + (go,)
                    hi = list(s.hi)
                    hi[r] = go
                    t = replace(s, issued=tuple(iss), hi=tuple(hi))
                    out.append(set_rank(t, r, n_iss=rk.n_iss + 1, snapped=False, contrib=False,
                                        pc="A"))        # `continue`
                else:
                    out.append(set_rank(s, r, pc=nxt))
            elif rk.pc == "E":
                out.append(set_rank(publish(s, r), r, pc=nxt))
            else:  # "F"
                if rk.n_iss > 0 and all(x >= rk.g + 1 for x in s.done):
                    t = publish(s, r)
                    out.append(set_rank(t, r, pub=rk.g, g=rk.g + 1, n_iss=rk.n_iss - 1, pc="A"))
                else:
                    out.append(set_rank(s, r, pc=nxt))
            if only_ctrl_of is not None:
                continue
            # workers of owner r finish the oldest round r issued
            if s.issued[r]:
                x = s.issued[r][0]
                iss = list(s.issued)
                iss[r] = iss[r][1:]
                done = list(s.done)
                done[r] = x + 1
                out.append(replace(s, issued=tuple(iss), done=tuple(done)))
            # host: post the next offer (back to back)
            if rk.next_offer < rounds:
                out.append(set_rank(s, r, queue=rk.queue + (rk.next_offer,),
                                    next_offer=rk.next_offer + 1))
            # host reader (ec_wait with pin): pin the latest published round,
            # wait for the acknowledgement, re-check, read, unpin
            if r == reader_rank:
                st = rk.reader
                if st[0] == "idle" and rk.host_done >= 1:
                    G = rk.host_done - 1
                    out.append(set_rank(s, r, pin=G, pin_seq=rk.pin_seq + 1,
                                        reader=("ack", G, rk.pin_seq + 1)))
                elif st[0] == "ack" and rk.acked >= st[2]:
                    G = st[1]
                    D = rk.host_done - 1
                    if D < G + R - rl:
                        out.append(set_rank(s, r, reader=("read", G)))
                    else:
                        out.append(set_rank(s, r, pin=D, pin_seq=rk.pin_seq + 1,
                                            reader=("ack", D, rk.pin_seq + 1)))
                elif st[0] == "read":
                    out.append(set_rank(s, r, pin=INF, pin_seq=rk.pin_seq + 1, reader=("done",)))
        return out

    def check(s: State):
        for r in range(p):
            rk = s.ranks[r]
            if rk.n_iss > lead:
                rep.violations.append(("too many rounds in flight", r, s))
            if rk.g > 0 and rk.host_done > rk.g:
                rep.violations.append(("published a round not completed", r, s))
            if rk.reader[0] == "read":
                G = rk.reader[1]
                # rounds are issued in order per owner: some X > G with
                # X = G mod R has written (or is writing) the slot iff an owner
                # issued a generation >= G + R
                if max(s.hi) >= G + R:
                    rep.violations.append(("pinned slot overwritten", r, G, max(s.hi), s))

    def core(s: State):
        return replace(s, ranks=tuple(replace(rk, pc="A") for rk in s.ranks))

    while stack:
        s = stack.pop()
        if s in seen:
            continue
        seen.add(s)
        if len(seen) > max_states:
            rep.violations.append(("state space exceeded", max_states))
            break
        check(s)
        if rep.violations:
            break
        succ = [x for x in successors(s) if x != s]
        terminal = all(rk.next_offer == rounds and not rk.queue and rk.n_iss == 0 and
                       rk.g == rounds and rk.pub < 0 for rk in s.ranks) and \
            all(not q for q in s.issued)
        if terminal:
            rep.terminals += 1
            continue
        # controller sections that change nothing only advance pc: stuck means
        # no host / worker action is enabled and no rank's full controller
        # cycle (its six sections in order) changes anything but pc
        c0 = core(s)
        if all(core(x) == c0 for x in succ):
            moved = False
            for r in range(p):
                t = s
                for _ in range(6):
                    t = successors(t, only_ctrl_of=r)[0]
                    if core(t) != c0:
                        moved = True
                        break
                if moved:
                    break
            if not moved:
                rep.violations.append(("deadlock", s))
                break
        stack.extend(succ)
    rep.states = len(seen)
    return rep

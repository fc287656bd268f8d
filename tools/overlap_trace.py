"""Schedule checker for the static-group overlap (§III-C-2; SPEC.md scheduler
`validate_trace`). Host logic only: it reads times, it computes nothing of the method.

A trace of one step is
  * groups: ``Lars.groups()`` (k = 0 first in backward order; tensors first..last, flat span begin/len),
  * bwd_done: ``{tensor: ms}`` — when the producer finished writing each tensor's gradient,
  * lib: ``Lars.group_trace_read()`` — ready[k], rs_start[k], rs_end[k] per group and ``applied``,
all in ms on one clock (CUDA events relative to group 0's ready event).

Conditions (SPEC.md validate_trace (a)-(d)):
  (a) a group's reduction starts after every member's gradient is written;
  (b) reductions start in group order;
  (c) the step is applied after every reduction ended;
  (d) byte conservation: every tensor in exactly one group, the spans tile [0, padded) once.
"""
from __future__ import annotations

EPS_MS = 2e-3  # CUDA event resolution is ~0.5 us; allow a little more


def validate_trace(groups: list[dict], bwd_done: dict, lib: dict, n_tensors: int, padded: int,
                   eps: float = EPS_MS) -> list[str]:
    bad = []
    seen = {}
    for k, g in enumerate(groups):
        for l in range(g["first"], g["last"] + 1):
            if l in seen:
                bad.append(f"(d) tensor {l} in groups {seen[l]} and {k}")
            seen[l] = k
    missing = sorted(set(range(n_tensors)) - set(seen))
    if missing:
        bad.append(f"(d) tensors in no group: {missing[:8]}")
    spans = sorted((g["begin"], g["len"]) for g in groups)
    pos = 0
    for b, n in spans:
        if b != pos:
            bad.append(f"(d) span gap/overlap at element {pos} (next group begins at {b})")
        pos = b + n
    if pos != padded:
        bad.append(f"(d) spans cover {pos} elements, layout has {padded}")
    for k, g in enumerate(groups):
        members = [bwd_done[l] for l in range(g["first"], g["last"] + 1) if l in bwd_done]
        if members and lib["rs_start"][k] + eps < max(members):
            bad.append(f"(a) group {k} reduction started {max(members) - lib['rs_start'][k]:.4f} ms before its "
                       f"last member was written")
        if k and lib["rs_start"][k] + eps < lib["rs_start"][k - 1]:
            bad.append(f"(b) group {k} started before group {k - 1}")
    if lib["rs_end"] and lib["applied"] + eps < max(lib["rs_end"]):
        bad.append("(c) step applied before every reduction ended")
    return bad

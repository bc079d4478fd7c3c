"""Oracle verification: restates ``specpipe/verify.py`` (TEST INFRASTRUCTURE).

Records are any object with ``tokens``, ``min_pos``, ``max_pos``,
``logit_slots`` (pos -> row), ``seq_id``, ``kind``, ``status``, ``run_id``
and ``chain()``.
"""

from __future__ import annotations

from .model import greedy_sample


class OracleVerifyError(RuntimeError):
    pass


def verify_run(rec, rows, accepted, base_logits=None, eos_token=None):
    """Chain walk (``verify.py:43-124``).  Returns a dict with the
    VerifyResult fields."""
    acc = list(accepted)
    newly, examined = [], 0
    pred = None
    nxt, mismatch, end = None, False, rec.min_pos

    def row(p):
        if p not in rec.logit_slots:
            raise OracleVerifyError(f"no logits slot for position {p}")
        return rows[rec.logit_slots[p]]

    for i, tok in enumerate(rec.tokens):
        p = rec.min_pos + i
        if p < len(acc):
            if tok != acc[p]:
                raise OracleVerifyError("run contradicts accepted context")
            pred, end = row(p), p + 1
            continue
        if p != len(acc):
            raise OracleVerifyError("gap before frontier")
        if pred is None:
            if base_logits is None:
                raise OracleVerifyError("no predictor for frontier")
            pred = base_logits
        examined += 1
        want = greedy_sample(pred)
        if tok != want:
            nxt, mismatch = want, True
            break
        newly.append(tok)
        acc.append(tok)
        pred, end = row(p), p + 1
        if eos_token is not None and tok == eos_token:
            return dict(accepted=tuple(newly), n_accepted=len(newly),
                        next_token=None, terminal=True, examined=examined,
                        mismatch=False, matched_end=end)
    if not mismatch and nxt is None:
        last = rec.min_pos + len(rec.tokens) - 1
        if pred is not None and last + 1 == len(acc):
            nxt = greedy_sample(pred)
    terminal = eos_token is not None and nxt is not None and nxt == eos_token
    return dict(accepted=tuple(newly), n_accepted=len(newly), next_token=nxt,
                terminal=terminal, examined=examined, mismatch=mismatch,
                matched_end=end)


def detect_stale_runs(fifo, accepted):
    """(``verify.py:127-153``) -> list of (record, "invalid"|"superfluous")."""
    out = []
    last = len(accepted) - 1
    for rec in fifo:
        if rec.status != "in-flight":
            continue
        bad = rec.kind != "non-speculative" and any(
            p < len(accepted) and t != accepted[p] for p, t in rec.chain())
        if bad:
            out.append((rec, "invalid"))
        elif rec.max_pos < last:
            out.append((rec, "superfluous"))
    return out


def apply_acceptance(matched_end, rec, live):
    """Command list committing a verified run (``verify.py:156-178``)."""
    if rec.seq_id == 0:
        return []
    cmds = []
    if matched_end > rec.min_pos:
        cmds.append(("copy", (rec.seq_id,
                              tuple(sorted({0, *live} - {rec.seq_id})),
                              matched_end)))
    cmds.append(("remove", (rec.seq_id, 0)))
    return cmds

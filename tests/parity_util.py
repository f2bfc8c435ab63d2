"""Parity checker: compare the engine's index sequence with the oracle's
prefix-wise up to the first pivot step whose oracle margin (|best|-|second|)/|best| is at or
below the margin rule (1e-10 relative); beyond that only status and error are compared."""
import numpy as np

MARGIN_RULE = 1e-10


def margin(best, second):
    if second < 0 or best <= 0:
        return float("inf")
    return (best - second) / best


def compare_runs(oracle_run, factors, trace, rule=MARGIN_RULE):
    """Returns (verdict dict). `identical` is True when I and J agree on the pinned prefix."""
    o_steps = oracle_run.steps
    first_tie = None
    for q, (_, k, _, b, s) in enumerate(o_steps):
        if margin(b, s) <= rule:
            first_tie = q
            break
    # the pinned prefix in terms of accepted (I, J) entries: all blocks strictly before the
    # iteration that contains the first sub-margin step
    if first_tie is None:
        pinned_iters = len(oracle_run.rhos)
    else:
        pinned_iters = o_steps[first_tie][1]
    widths = oracle_run.widths[:pinned_iters]
    npin = int(sum(widths))
    I_o, J_o = oracle_run.row_indices[:npin], oracle_run.col_indices[:npin]
    I_e, J_e = factors.row_indices[:npin], factors.col_indices[:npin]
    return {
        "pinned_entries": npin,
        "first_sub_margin_step": first_tie,
        "identical": I_o == I_e and J_o == J_e,
        "full_identical": oracle_run.row_indices == factors.row_indices and
        oracle_run.col_indices == factors.col_indices,
        "status_equal": oracle_run.status == trace.status,
        "min_margin": min((margin(b, s) for (_, _, _, b, s) in o_steps), default=float("inf")),
    }

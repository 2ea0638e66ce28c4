"""Decoder for the canonical state snapshot,
shared by the reference driver (oracle/ref_driver.cpp), the C oracle and the
product (econo_snapshot)."""
import numpy as np

REQ_FIELDS = ["state", "generated", "predicted_rl", "padded_rl", "allowance", "generated_at_epoch",
              "occupied_kvc", "hosted", "was_preempted", "preempt_count", "reserve_draws",
              "alloc_failure", "prefill_done", "waiting_time", "preemption_time", "execution_time",
              "dispatch_time", "first_token_time", "completion_clock", "last_enqueue_time",
              "sched_share", "penalty_extra", "slo_deadline"]
FLOAT_FIELDS = set(REQ_FIELDS[13:])


def _f(v):
    return np.int64(v).view(np.float64).item()


def decode(w):
    w = [int(x) for x in w]
    p = 0

    def take(k=1):
        nonlocal p
        out = w[p:p + k]
        p += k
        return out if k > 1 else out[0]

    assert take() == 0x45434F4E, "bad snapshot magic"
    d = {}
    (d["iter"], clk, d["completed"], d["arrival_cursor"], d["free_tokens"], d["reserved_used"],
     d["written_total"], d["hosted_total"], d["hosted_overruns"], d["exam_count"], n) = take(11)
    d["clock"] = _f(clk)
    d["n"] = n
    d["pt_queue"] = [take() for _ in range(take())]
    groups = []
    for _ in range(take()):
        g = dict(zip(["group_id", "padded_rl", "formed_at", "min_deadline", "max_occupied",
                      "key_deadline", "key_kvc", "key_length", "key_seq"], take(9)))
        g["formed_at"] = _f(g["formed_at"])
        g["min_deadline"] = _f(g["min_deadline"])
        g["members"] = [take() for _ in range(take())]
        groups.append(g)
    d["gt_groups"] = groups
    d["slots"] = [dict(zip(["host_id", "hosted_id", "start_offset", "length", "deadline_usage",
                            "abs_start"], take(6))) for _ in range(take())]
    hold = {}
    for _ in range(take()):
        rid, total, nr = take(3)
        regs = [tuple(take(2)) for _ in range(nr)]
        hold[rid] = dict(total=total, regions=regs)
    d["holdings"] = hold
    d["free"] = [tuple(take(2)) for _ in range(take())]
    d["reserved"] = dict(tuple(take(2)) for _ in range(take()))
    d["written"] = dict(tuple(take(2)) for _ in range(take()))
    d["running"] = [take() for _ in range(take())]
    reqs = []
    for _ in range(n):
        vals = take(len(REQ_FIELDS))
        r = {k: (_f(v) if k in FLOAT_FIELDS else v) for k, v in zip(REQ_FIELDS, vals)}
        reqs.append(r)
    d["requests"] = reqs
    if p < len(w):  # baseline-policy tail
        assert take() == 0x42415345, "bad baseline tail magic"
        d["decode_pause"], d["admission_open"], stall = take(3)
        d["pending_stall"] = _f(stall)
        d["admit_order"] = [take() for _ in range(take())]
        d["ongoing_prefills"] = [take() for _ in range(take())]
        for r in reqs:
            r["prefill_target"] = take()
    assert p == len(w), "trailing words in snapshot"
    return d

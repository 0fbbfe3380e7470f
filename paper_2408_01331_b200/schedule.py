"""Slice plans accepted by the Trainer (src/schedule.py:22-131, compact).

Policy ordering is outside the hot path: the B200 trainer runs every live
job in lockstep, so a plan only says which (job, epoch) slices exist.
These helpers build the same slice lists as the reference planners so a
plan object can be passed exactly as before; the reference's own
SchedulePlan is accepted too (duck-typed on ``policy`` / ``slices``).
"""
from __future__ import annotations

from dataclasses import dataclass

POLICIES = ("fcfs", "priority", "sjf", "rr")


@dataclass(frozen=True)
class Slice:
    job_id: str
    epoch: int


@dataclass(frozen=True)
class SchedulePlan:
    policy: str
    slices: tuple

    def __len__(self):
        return len(self.slices)

    def job_ids(self) -> list:
        out = []
        for s in self.slices:
            if s.job_id not in out:
                out.append(s.job_id)
        return out

    def completion_index(self, job_id: str) -> int:
        for i in range(len(self.slices) - 1, -1, -1):
            if self.slices[i].job_id == job_id:
                return i + 1
        raise KeyError(job_id)

    def without(self, job_id: str, executed: int) -> "SchedulePlan":
        keep = tuple(s for s in self.slices[executed:] if s.job_id != job_id)
        return SchedulePlan(self.policy, self.slices[:executed] + keep)


def _run_to_end(jobs):
    return [Slice(j.job_id, e) for j in jobs for e in range(j.completed_epochs, j.hypers.epochs)]


def _round_robin(jobs):
    nxt = {j.job_id: j.completed_epochs for j in jobs}
    live = [j for j in jobs if nxt[j.job_id] < j.hypers.epochs]
    out = []
    while live:
        still = []
        for j in live:
            out.append(Slice(j.job_id, nxt[j.job_id]))
            nxt[j.job_id] += 1
            if nxt[j.job_id] < j.hypers.epochs:
                still.append(j)
        live = still
    return out


def make_plan(policy: str, jobs: list, sjf_metric: str = "epochs") -> SchedulePlan:
    if not jobs:
        raise ValueError("cannot plan an empty job list")
    if len({j.job_id for j in jobs}) != len(jobs):
        raise ValueError("duplicate job ids in plan input")
    by_arrival = sorted(jobs, key=lambda j: j.arrival_seq)
    if policy == "fcfs":
        return SchedulePlan("fcfs", tuple(_run_to_end(by_arrival)))
    if policy == "rr":
        return SchedulePlan("rr", tuple(_round_robin(by_arrival)))
    if policy == "priority":
        out = []
        for prio in sorted({j.priority for j in jobs}):
            out += _round_robin(sorted((j for j in jobs if j.priority == prio), key=lambda j: j.arrival_seq))
        return SchedulePlan("priority", tuple(out))
    if policy == "sjf":
        if sjf_metric == "size":
            from .engine import param_count

            key = {j.job_id: param_count(j.graph) for j in jobs}
        elif sjf_metric == "epochs":
            key = {j.job_id: j.hypers.epochs for j in jobs}
        else:
            raise ValueError(f"sjf metric must be one of ('size', 'epochs'), got {sjf_metric!r}")
        return SchedulePlan("sjf", tuple(_run_to_end(sorted(jobs, key=lambda j: (key[j.job_id], j.arrival_seq)))))
    raise ValueError(f"policy must be one of {POLICIES}, got {policy!r}")

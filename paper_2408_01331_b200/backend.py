"""Backend switch: run the reference's Workspace / CLI on the B200 hot path.

The reference's end-to-end workflow (hybridnn.workspace.Workspace.run, src/workspace.py:220-340,
and the CLI over it, src/cli.py) reaches the training path through five module-level names of
hybridnn.workspace: ``unify_jobs`` (merge + checkpoint restore, :412-422), ``Trainer``,
``separate`` / ``package`` (the separator thread, :271-285) and ``Checkpoint`` / ``restore_checkpoint``
(pause sink and resume, :200-216, :300-311).  :func:`install` rebinds exactly those names to this
package, so queue handling, dataset store, reports and the memory model stay the reference's own
and every training step runs on the grouped sm_100a kernels::

    import hybridnn
    from paper_2408_01331_b200 import backend
    backend.install(hybridnn)            # or: python -m paper_2408_01331_b200.backend <hybridnn CLI args>
    hybridnn.Workspace(root).run("rr")

:func:`uninstall` restores the reference's bindings.  The reference objects the Workspace passes
in (TrainingJob, ModelGraph, HyperParams, Dataset, SchedulePlan) are accepted as they are
(TrainingJob.coerce, duck-typed datasets and plans).
"""
from __future__ import annotations

import sys

ROUTED = ("unify_jobs", "Trainer", "separate", "package", "Checkpoint", "restore_checkpoint")


def unify_jobs(jobs, records, root):
    """merge(), then restore every checkpointed job into the fresh hybrid (src/workspace.py:412-422)."""
    from .train import Checkpoint, restore_checkpoint
    from .unify import merge

    hybrid = merge(jobs)
    for job in jobs:
        rec = records[job.job_id]
        if rec.get("checkpoint") and job.completed_epochs > 0:
            restore_checkpoint(hybrid, Checkpoint.decode((root / rec["checkpoint"]).read_bytes()))
    return hybrid


def _workspace_module(hybridnn):
    import importlib

    return importlib.import_module(hybridnn.__name__ + ".workspace")


def install(hybridnn) -> dict:
    """Point hybridnn.workspace's training path at this package; returns the replaced bindings."""
    from .separate import package, separate
    from .train import Checkpoint, Trainer, restore_checkpoint

    ws = _workspace_module(hybridnn)
    ours = {"unify_jobs": unify_jobs, "Trainer": Trainer, "separate": separate, "package": package,
            "Checkpoint": Checkpoint, "restore_checkpoint": restore_checkpoint}
    saved = ws.__dict__.get("_hnn_b200_saved")
    if saved is None:
        saved = {name: getattr(ws, name) for name in ROUTED}
        ws._hnn_b200_saved = saved
    for name in ROUTED:
        setattr(ws, name, ours[name])
    return saved


def uninstall(hybridnn) -> None:
    ws = _workspace_module(hybridnn)
    saved = ws.__dict__.pop("_hnn_b200_saved", None)
    if saved:
        for name, value in saved.items():
            setattr(ws, name, value)


def installed(hybridnn) -> bool:
    from .train import Trainer

    return _workspace_module(hybridnn).Trainer is Trainer


def main(argv=None) -> int:
    """``python -m paper_2408_01331_b200.backend ARGS``: the reference CLI with the B200 backend."""
    import hybridnn
    from hybridnn import cli

    install(hybridnn)
    try:
        cli.main(args=list(sys.argv[1:] if argv is None else argv), prog_name="hybridnn")
    except SystemExit as exc:  # the reference CLI's exit codes (0 ok, 2 validation, ...) pass through
        return int(exc.code or 0)
    return 0


if __name__ == "__main__":
    sys.exit(main())

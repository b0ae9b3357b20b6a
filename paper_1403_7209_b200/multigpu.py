"""Owner-compute multi-GPU execution (one process per GPU) — under construction.

See DESIGN.md §6.  Until the NCCL halo layer lands, multi-rank execution
raises instead of silently running something else.
"""
from __future__ import annotations

from .core import ExecError


def run_program_distributed(program, mesh, config):
    raise ExecError("multi-GPU execution (nranks > 1) is not implemented yet")


def bench_distributed(args, metric):
    raise ExecError("multi-GPU bench is not implemented yet")

"""absim-bench output schema (tools/bench_main.cpp:24-28, 384-434) for runs
of this engine, so results drop into the reference's sweep tooling.

`options` carries the bench's run options (model, agents, iterations,
threads, domain_count, env, allocator, sorting_frequency, static_detection,
seed); for a device run `threads` is the number of GPUs, `domain_count` the
number of slabs and `allocator` "device_pool". `report` is a
SimulationReport (Simulation.phase_report()).
"""
from __future__ import annotations

from dataclasses import dataclass

CSV_HEADER = ("model,agents,iterations,threads,domain_count,env,allocator,sorting_freq,"
              "static_detect,wall_ms_total,wall_ms_agent_ops,wall_ms_env_update,"
              "wall_ms_sorting,wall_ms_setup_teardown,peak_rss_bytes,force_evals,"
              "repetition")


@dataclass
class RunOptions:
    model: str = "clustering"
    agents: int = 1000
    iterations: int = 10
    threads: int = 1
    domain_count: int = 1
    env: str = "uniform_grid"
    allocator: str = "device_pool"
    sorting_frequency: int = 0
    static_detection: bool = False
    seed: int = 42


def csv_row(o: RunOptions, r, repetition: int = 0) -> str:
    """One row under CSV_HEADER (bench_main.cpp:384-396: fixed, 3 decimals)."""
    f = lambda v: f"{v:.3f}"  # noqa: E731
    return ",".join([o.model, str(o.agents), str(o.iterations), str(o.threads), str(o.domain_count), o.env,
                     o.allocator, str(o.sorting_frequency), "1" if o.static_detection else "0",
                     f(r.total_wall_ms), f(r.agent_ops_ms), f(r.env_update_ms), f(r.sorting_ms),
                     f(r.setup_teardown_ms), str(r.peak_rss_bytes), str(r.force_evaluations), str(repetition)])


def report_json(o: RunOptions, r) -> dict:
    """bench_main.cpp:398-434 report_to_json."""
    rep = {
        "iterations": r.iterations,
        "final_agent_count": r.final_agent_count,
        "wall_ms_total": r.total_wall_ms,
        "wall_ms_agent_ops": r.agent_ops_ms,
        "wall_ms_env_update": r.env_update_ms,
        "wall_ms_sorting": r.sorting_ms,
        "wall_ms_setup_teardown": r.setup_teardown_ms,
        "peak_rss_bytes": r.peak_rss_bytes,
        "force_evaluations": r.force_evaluations,
        "force_skips": r.force_skips,
        "agents_added": r.agents_added,
        "agents_removed": r.agents_removed,
        "agents_sorted": r.agents_sorted,
        "same_domain_steals": r.same_domain_steals,
        "cross_domain_steals": r.cross_domain_steals,
        "allocator_batch_migrations": r.allocator_batch_migrations,
        "per_operation_ms": dict(r.per_operation_ms),
        "per_iteration_ms": list(r.per_iteration_ms),
    }
    return {"model": o.model, "agents": o.agents, "iterations": o.iterations, "threads": o.threads,
            "domain_count": o.domain_count, "env": o.env, "allocator": o.allocator,
            "sorting_frequency": o.sorting_frequency, "static_detection": o.static_detection,
            "seed": o.seed, "report": rep}

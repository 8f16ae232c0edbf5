"""CPU: the C-ABI library loads and exports every symbol include/absim_gpu.h
declares; without a GPU, context creation fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "absim_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(abs_gpu_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol(engine):
    from paper_2301_06984_b200 import _native as N
    lib = N.load()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(N.EXPORTS) == declared


def test_library_is_sm100a(engine):
    from paper_2301_06984_b200 import _native as N
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {N.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu(engine):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2301_06984_b200 import _native as N
    with pytest.raises(N.AbsimError) as e:
        engine.Simulation(engine.SimulationParams())
    assert e.value.code == N.ABS_ERR_NO_DEVICE


def test_params_validation_mirrors_reference(engine):
    # params.cpp:44-72 — raised before any device work
    for kw in (dict(simulation_time_step=0.0), dict(max_displacement=0.0),
               dict(repulsion_coefficient=-1.0), dict(force_threshold=-1.0),
               dict(fixed_box_length=-1.0)):
        with pytest.raises(ValueError):
            engine.Simulation(engine.SimulationParams(**kw))


def test_models_header_compiles_as_c(tmp_path):
    """absim_models.h is shared verbatim by C (oracle), C++ (harness) and CUDA."""
    src = tmp_path / "t.c"
    src.write_text('#include "absim_models.h"\n#include "absim_gpu.h"\n'
                   "int main(void){ return abs_rng_word(1,2,3) == 0; }\n")
    rc = os.system(f"gcc -std=c11 -I{ROOT}/include {src} -o {tmp_path}/t -lm")
    assert rc == 0


def test_report_schema_matches_reference_bench():
    """CSV header / JSON keys of tools/bench_main.cpp:24-28, 398-434."""
    from paper_2301_06984_b200 import report as R
    from paper_2301_06984_b200.engine import SimulationReport
    r = SimulationReport(iterations=3, final_agent_count=10, force_evaluations=7, total_wall_ms=1.5)
    o = R.RunOptions(model="clustering", agents=10, iterations=3)
    row = R.csv_row(o, r, 2)
    assert len(row.split(",")) == len(R.CSV_HEADER.split(","))
    assert row.startswith("clustering,10,3,1,1,uniform_grid,device_pool,0,0,1.500,")
    j = R.report_json(o, r)
    assert set(j) == {"model", "agents", "iterations", "threads", "domain_count", "env", "allocator",
                      "sorting_frequency", "static_detection", "seed", "report"}
    assert {"wall_ms_total", "per_iteration_ms", "per_operation_ms", "force_evaluations",
            "allocator_batch_migrations"} <= set(j["report"])

"""Config 5 / SURVEY.md §8(f) rank 1: the reference simulator relinked with the
GPU adapter (integration/aragog_gpu.cpp) -- ConfigPredictor::predict,
beam_schedule, enumerate_members and select_per_input_config on the B200 --
must produce byte-identical JSONL traces to the unmodified reference build
(the criterion-8 determinism contract, tests/acceptance/criteria.cpp:367-419),
and the reference acceptance criteria must all pass on the GPU build."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = os.path.join(ROOT, "integration", "_build")
SC = os.path.join(B, "proj", "scenarios")

pytestmark = pytest.mark.gpu

need = pytest.mark.skipif(not os.path.exists(os.path.join(B, "sim_trace_gpu")),
                          reason="integration/_build not built (needs /root/reference at build time)")


def _run(binary, scenario, policy, out, *opts):
    r = subprocess.run([os.path.join(B, binary), os.path.join(SC, scenario), policy, out, *opts],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])


@need
@pytest.mark.parametrize("scenario", ["reference.json", "reference_noisy.json", "mm1.json",
                                      "decompose.json"])
@pytest.mark.parametrize("policy", ["aragog", "per-workflow", "per-input-static",
                                    "per-input-runtime-cost"])
def test_trace_byte_identical(tmp_path, scenario, policy):
    ref = str(tmp_path / "ref.jsonl")
    gpu = str(tmp_path / "gpu.jsonl")
    a = _run("sim_trace_ref", scenario, policy, ref, "--requests", "120")
    b = _run("sim_trace_gpu", scenario, policy, gpu, "--requests", "120")
    assert b["gpu_launches"] > 0, "the GPU build ran no kernels"
    assert a["rounds"] == b["rounds"] and a["completed"] == b["completed"]
    assert open(ref, "rb").read() == open(gpu, "rb").read()


@need
def test_trace_byte_identical_horizon_sweep_point(tmp_path):
    # a loaded Poisson point of the shipped sweep (reference.json rates 0.5..3.5)
    ref = str(tmp_path / "ref.jsonl")
    gpu = str(tmp_path / "gpu.jsonl")
    _run("sim_trace_ref", "reference.json", "aragog", ref, "--horizon", "120", "--rate", "3.0")
    b = _run("sim_trace_gpu", "reference.json", "aragog", gpu, "--horizon", "120", "--rate", "3.0")
    assert b["gpu_launches"] > 0
    assert open(ref, "rb").read() == open(gpu, "rb").read()


@need
def test_acceptance_criteria_on_gpu_build():
    r = subprocess.run([os.path.join(B, "acceptance_gpu"), "--jobs", "4"], capture_output=True,
                       text=True, timeout=1200)
    lines = [l for l in r.stdout.splitlines() if l.startswith("criterion")]
    assert len(lines) == 10, r.stdout + r.stderr
    assert all(" PASS " in l for l in lines), "\n".join(lines)
    assert r.returncode == 0

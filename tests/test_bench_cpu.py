"""CPU: bench.py's reference arm (the reference's own DecoupledTrainer::step from oracle/_ref on
the host) prints one valid JSON line with the contract's keys, and the FLOP model matches
SURVEY §8d."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_flop_model_matches_survey():
    import bench
    # C2 7.255 GFLOP / image, C5 463.9 GFLOP / image
    assert abs(bench.flops_per_image(bench.CONFIGS["C2"]) / 1e9 - 7.255) < 0.005
    assert abs(bench.flops_per_image(bench.CONFIGS["C5"]) / 1e9 - 463.9) < 0.1


def test_kappa_step_is_scaled_to_the_stage_size():
    import bench
    import paper_2009_01462_b200  # noqa: F401  (StepParams)
    for name in ("C2", "C5"):
        cfg = bench.CONFIGS[name]
        sp = bench.step_params(cfg)
        n = cfg["B"] * cfg["h"] * cfg["w"] * cfg["c"]
        assert abs(sp.kappa_lr * n / (2 * sp.beta) - bench.KAPPA_STEP) < 1e-12 * bench.KAPPA_STEP + 1e-20


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "librespar_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-images", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0

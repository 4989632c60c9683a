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


def test_reference_labels_follow_the_reference_rng():
    """bench's synthetic labels are the reference's next_u64() % 10 after the pixel draws
    (acceptance.cpp:69-73 pattern), checked against the oracle's splitmix64 stream."""
    import bench
    from oracle import respar_oracle as O
    rng = O.Rng(1234)
    rng.next_u64_block(300)                      # the pixels
    want = [int(v) % 10 for v in rng.next_u64_block(17)]
    assert bench.reference_labels(1234, 300, 17) == want


def test_gpus_flag_must_match_the_world_size():
    env = {**os.environ, "WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--plan"], env=env,
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


def test_gpus_flag_spawns_one_rank_per_gpu():
    """--gpus 4 without torchrun re-launches itself under torch.distributed.run (127.0.0.1):
    every rank reports its stages (C3: K = 8 -> two per rank) and neighbours."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--plan"], env=env,
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = sorted((json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")), key=lambda d: d["rank"])
    assert [d["stages"] for d in lines] == [[0, 2], [2, 4], [4, 6], [6, 8]]
    assert [d["prev_rank"] for d in lines] == [None, 0, 1, 2]
    assert [d["next_rank"] for d in lines] == [1, 2, 3, None]
    assert all(d["world"] == 4 for d in lines)

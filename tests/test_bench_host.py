"""bench.py host logic without a GPU: the strong-scaling shard plan (SURVEY
§8e) tiles every config exactly, both arms print the same config dict, and
`--gpus 2` starts two ranks itself (world-size-2 gloo run of the reference
arm, which needs no device)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("idx", sorted(bench.CONFIGS))
def test_strong_shards_tile_the_config(idx, world):
    cfg = bench.CONFIGS[idx]
    shares = [bench.local_config(cfg, r, world, "strong") for r in range(world)]
    label = bench.scaling_label(cfg, world, "strong")
    f_total = bench.work_of(cfg)[0]
    f_sum = sum(bench.work_of(c)[0] for c in shares)
    if label == "weak":  # cfg1: replicas
        assert cfg["dtype"] == "f32"
        assert all(c == dict(cfg, split_kv=False) for c in shares)
        return
    assert f_sum == pytest.approx(f_total, rel=1e-12)  # no unit dropped or duplicated
    pat = cfg["pattern"]
    if pat in bench.GRAN:
        assert all(c["M"] % bench.GRAN[pat] == 0 for c in shares)
    if pat == "attention" and cfg["Sq"] == 1 and world > 1:
        assert all(c["split_kv"] and c["Skv"] * world == cfg["Skv"] for c in shares)
        assert all(c["segments_global"] % world == 0 for c in shares)


def test_weak_scaling_gives_every_rank_the_config():
    cfg = bench.CONFIGS[1]
    for r in range(4):
        assert bench.local_config(cfg, r, 4, "weak") == dict(cfg, split_kv=False)


def test_both_arms_print_the_same_config():
    for idx, cfg in bench.CONFIGS.items():
        for world in (1, 8):
            a = bench.config_dict(cfg, world, "strong")
            assert a == bench.config_dict(dict(cfg), world, "strong")
            assert a["workload"] == cfg["name"]
            assert "kernel" not in a  # implementation details live in impl_detail


def test_parallelism_names_the_split():
    assert "split-KV" in bench.parallelism(bench.CONFIGS[2], 8, "strong")
    assert "batch/head" in bench.parallelism(bench.CONFIGS[1], 8, "strong")
    assert "tokens" in bench.parallelism(bench.CONFIGS[3], 8, "strong")
    assert "replicas" in bench.parallelism(bench.CONFIGS[0], 8, "strong")


@pytest.mark.skipif(not os.path.exists(bench.REF_DRIVER), reason="oracle/_ref not built")
def test_gpus_2_launches_two_ranks_and_rank0_prints_one_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--config", "0", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={k: v for k, v in os.environ.items()
                            if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"] == bench.config_dict(bench.CONFIGS[0], 2, "strong")
    assert line["extrapolated_from_rows"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def _gloo_worker():
    """Runs inside each torchrun rank (see the test below)."""
    import torch

    D = bench.Dist("gloo")
    assert D.world == 2 and D.dev.type == "cpu"
    # max over ranks
    assert D.max(float(D.rank + 1)) == 2.0
    # sequence all-gather in rank (= slice) order
    t = torch.full((3, 4, 2), float(D.rank))
    g = D.gather_seq(t)
    assert g.shape == (3, 8, 2) and g[:, :4].eq(0).all() and g[:, 4:].eq(1).all()
    # shard ranges of cfg2 / cfg4 agree across ranks and cover the config
    objs = D.gather_objects({k: bench.local_config(bench.CONFIGS[k], D.rank, 2, "strong")
                             for k in (1, 3)})
    assert sum(o[1]["H"] for o in objs) == 256 and sum(o[3]["M"] for o in objs) == 8192
    merged = bench.merge_parity([{"rows_checked": 3, "pass": True, "max_scaled_err": {"d1": 1e-3}},
                                 {"rows_checked": 5, "pass": True, "max_scaled_err": {"d1": 2e-3}}])
    assert merged["rows_checked"] == 8 and merged["max_scaled_err"]["d1"] == 2e-3
    D.close()
    print("gloo-ok", D.rank)


def test_dist_plumbing_world_size_2_gloo(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(f"import sys; sys.path.insert(0, {ROOT!r})\n"
                      "from tests.test_bench_host import _gloo_worker\n_gloo_worker()\n")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29613",
                        str(script)], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.count("gloo-ok") == 2

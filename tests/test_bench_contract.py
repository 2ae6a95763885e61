"""bench.py's multi-rank partition (CPU, -m "not gpu"): BASELINE configs[2] is a
batch of 64 pages sharded across 1/2/4/8 GPUs and configs[4]'s batch of 32
pages sharded across 8 -- strong scaling by default, every page on exactly
one rank; weak scaling (every rank a whole batch) only on request."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("P,world", [(64, 1), (64, 2), (64, 4), (64, 8), (32, 8), (32, 3), (5, 8)])
def test_strong_scaling_shards_the_batch(bench, P, world):
    got = [bench.page_shard(P, r, world, "strong") for r in range(world)]
    nxt = 0
    for first, n in got:
        assert first == nxt
        nxt += n
    assert nxt == P                                          # every page exactly once
    assert max(n for _, n in got) - min(n for _, n in got) <= 1


def test_weak_scaling_is_opt_in(bench):
    assert [bench.page_shard(64, r, 4, "weak") for r in range(4)] == [(0, 64), (64, 64), (128, 64), (192, 64)]
    import argparse
    ap = argparse.ArgumentParser()
    # the default of the real parser
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert '"--scaling", choices=["weak", "strong"], default="strong"' in src


def test_configs_match_baseline(bench):
    assert bench.CONFIGS[3][:3] == (64, 7016, 4960)
    assert bench.CONFIGS["5b"][:5] == (32, 4096, 4096, 51, 51)
    assert bench.cfg_key("5b") == "5b" and bench.cfg_key("3") == 3
    assert bench.SWEEP == (15, 31, 63, 127, 255)

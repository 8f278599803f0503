"""A fixed block of the differential fuzzer's seeds (tests/fuzz_cases.py): random sizes, kernels
and scene mutations, bin / forward / backward against the oracle by the bars of
tests/test_gpu_rasterizer.py."""
import pytest

import fuzz_cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("block", range(4))
def test_fuzz_block(ctx, port, block, capsys):
    failed = [seed for seed in range(100 * block, 100 * block + 100) if not fuzz_cases.trial(ctx, port, seed)]
    assert not failed, (failed, capsys.readouterr().out[-2000:])


@pytest.mark.parametrize("block", range(2))
def test_fuzz_chain_block(ctx, port, darbs, block, capsys):
    """The 3-D chain of one view (fit3d.cpp:108-159) on random cameras, scenes, kernels and losses."""
    failed = [seed for seed in range(100 * block, 100 * block + 100) if not fuzz_cases.chain_trial(ctx, port, darbs, seed)]
    assert not failed, (failed, capsys.readouterr().out[-2000:])


def test_fuzz_loss_block(ctx, port, capsys):
    """loss_total (loss.cpp:173-230) on random sizes, lambdas and image pairs."""
    failed = [seed for seed in range(200) if not fuzz_cases.loss_trial(ctx, port, seed)]
    assert not failed, (failed, capsys.readouterr().out[-2000:])


def test_fuzz_bins_block(ctx, port, capsys):
    """bin_splats on large and degenerate tile grids (32-bit tile keys, strips, K in the millions)."""
    failed = [seed for seed in range(40) if not fuzz_cases.bins_trial(ctx, port, seed)]
    assert not failed, (failed, capsys.readouterr().out[-2000:])

"""SPEC's transfer-time formula and the alpha-beta fit (CPU only)."""
import pytest

from paper_2504_09285_b200.model import fit_alpha_beta, transfer_time_ms


def test_spec_worked_example():
    # 16-token chunk, 131072 B/token, 25e6 B/ms, 0.05 ms latency -> 0.1339 ms
    assert transfer_time_ms(16, 131072, 25e6, 0.05) == pytest.approx(0.133886, abs=5e-7)
    assert round(transfer_time_ms(16, 131072, 25e6, 0.05), 4) == 0.1339


def test_zero_tokens_and_linearity():
    assert transfer_time_ms(0, 131072, 25e6, 0.05) == 0.0
    a = transfer_time_ms(100, 2048, 1e6, 0.0)
    assert transfer_time_ms(200, 2048, 1e6, 0.0) == pytest.approx(2 * a)


def test_fit_recovers_exact_parameters():
    xs = [2 ** k * 1e6 for k in range(10)]
    ys = [0.004 + x / 3.2e9 for x in xs]
    alpha, beta = fit_alpha_beta(xs, ys)
    assert alpha == pytest.approx(0.004, rel=1e-9) and beta == pytest.approx(3.2e9, rel=1e-9)

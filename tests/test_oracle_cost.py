"""Pins for the multiplication-count formulas of Appendix A.1 (tests/golden/cost_formulas.txt)."""
from math import comb

import oracle


def test_special_cases_printed_in_paper():
    for d in range(1, 12):
        assert oracle.fused_cost(d, 1) == 0 == oracle.conventional_cost(d, 1)
        assert oracle.fused_cost(d, 2) == d + d * d
        assert oracle.conventional_cost(d, 2) == d + comb(d + 1, 2) + d * d
    for N in range(1, 12):
        tri = sum(k - 1 for k in range(1, N + 1))
        assert oracle.fused_cost(1, N) == (N - 1) + tri
        assert oracle.conventional_cost(1, N) == 2 * (N - 1) + tri


def test_closed_forms_match_sums():
    """eq-fusedresulttwo and the lower bound eq-conventionaltwo, d >= 2."""
    for d in range(2, 10):
        for N in range(3, 10):
            F = (d ** (N + 2) - d ** 3 - (N - 1) * d ** 2 + (N - 1) * d)
            assert F % (d - 1) ** 2 == 0
            assert oracle.fused_cost(d, N) == F // (d - 1) ** 2
            low = ((N - 1) * d ** (N + 2) - N * d ** (N + 1) + d ** 2) // (d - 1) ** 2
            assert oracle.conventional_cost(d, N) >= low


def test_uniform_bound_including_special_case():
    """F(d,N) <= C(d,N) for all 1 <= d, N <= 10; (2,3) checked through eq-poly."""
    for d in range(1, 11):
        for N in range(1, 11):
            assert oracle.fused_cost(d, N) <= oracle.conventional_cost(d, N)
    d, N = 2, 3
    assert 0 <= d ** (N + 1) * (d * (N - 2) - N) + d * (d * d + N * (d * d - 1) + 1)


def test_benchmark_config_costs():
    """Per-config constants used for the FLOP numerators."""
    assert oracle.fused_cost(4, 4) == 444
    assert oracle.fused_cost(8, 5) == 42784
    assert oracle.fused_cost(6, 4) == 1854
    assert oracle.fused_cost(4, 7) == 29112
    assert oracle.fused_cost(3, 6) == 1626
    assert oracle.fused_cost(8, 4) == 5336

"""The barrier-free Kahn levelizer (HF_KAHN_ASYNC=1, levelize.cu k_lev_kahn_async)
under the same levelization parity tests as the default frontier-round Kahn:
the paper's worked graphs, C1 / scaled and full C3 / C5,
the three C2 shapes at 1M, tiny random DAGs, and cycles with their exact never-ready
counts (reading R8).  Levels, level_ptr and order bit-exact against the oracle."""
import pytest

import test_gpu_parity as P

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900, method="thread")]

hf = P.hf   # the module-scoped library fixture


@pytest.fixture(autouse=True)
def _kahn_async(monkeypatch):
    monkeypatch.setenv("HF_KAHN_ASYNC", "1")


test_golden_graphs = P.test_golden_graphs
test_config_single = P.test_config_single
test_config_single_full = P.test_config_single_full
test_c2_levelize_full = P.test_c2_levelize_full
test_tiny_random_dags = P.test_tiny_random_dags
test_cycles_reported_with_unready_count = P.test_cycles_reported_with_unready_count
test_cycle_in_large_graph = P.test_cycle_in_large_graph
test_empty_graph = P.test_empty_graph
test_isolated_nodes_and_negative_zero = P.test_isolated_nodes_and_negative_zero

"""Device unit tests of the EFT primitives (tests/native/devtests.cu), bitwise on the B200:
the ordered-FastTwoSum TwoSum equals Knuth's TwoSum and is exact; the AccuDOP renormalisation
as a FastTwoSum equals Knuth's TwoSum (cancelling quadruples included); the high-word sign and
zero tests equal the double comparisons; the shared-reciprocal
division and the fast-path sqrt equal __ddiv_rn / __dsqrt_rn whenever their guards pass."""
import ctypes

import pytest

torch = pytest.importorskip("torch")
from paper_2510_09892_b200._build import build_devtests  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_primitives_bitwise_on_device(seed):
    lib = ctypes.CDLL(build_devtests())
    lib.sgi_devtest.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
    out = torch.zeros(10, dtype=torch.int64, device="cuda")
    n = 1 << 24
    assert lib.sgi_devtest(seed, n, ctypes.c_void_p(out.data_ptr())) == 0
    c = out.cpu().tolist()
    assert c[0] == 0, f"two_sum value mismatches: {c}"
    assert c[2] == 0, f"two_sum not exact: {c}"
    assert c[3] == 0, f"div mismatches: {c}"
    assert c[5] == 0, f"sqrt mismatches: {c}"
    assert c[7] == 0, f"AccuDOP renormalisation: FastTwoSum != TwoSum: {c}"
    assert c[8] > n // 64, f"too few cancelling AccuDOP cases exercised: {c}"
    assert c[9] == 0, f"is_zero/is_pos/is_neg/is_nonneg != double comparisons: {c}"
    # the guards do fire on the tiny numerators / radicands the test feeds on purpose
    assert c[4] > 0 and c[6] > 0

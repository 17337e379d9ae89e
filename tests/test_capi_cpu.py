"""CPU-side checks of the product library: it loads without a GPU, exports every
symbol include/etune_cuda.h declares, and refuses to run without an sm_100 device
(no CPU fallback)."""
import ctypes as C

import pytest

from paper_2411_18873_b200 import capi


def test_exports_every_header_symbol():
    L = capi.lib()
    names = capi.header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_abi_version_and_defaults():
    assert capi.lib().etune_cu_abi_version() == 2
    d = capi.default_device_config()
    assert d.num_sms == 108 and d.constant_power_w == 60.0 and d.rng_seed == 1234  # device.hpp:17-36


def test_no_cpu_fallback():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = capi.lib().etune_cu_ctx_create(0, None, C.byref(h))
    assert st == 66  # ETUNE_ERR_NO_DEVICE


def test_status_codes_match_oracle_and_reference_order():
    # errors.hpp:15-100 declaration order == status 1..15 (oracle/ref_shim.cpp uses the same map)
    assert [capi.STATUS_NAMES[i] for i in range(1, 16)] == [
        "ParseError", "ValidationError", "SpaceExhausted", "IllegalSchedule", "TooLarge",
        "NonPositiveEnergy", "InsufficientData", "SchemaMismatch", "VersionMismatch", "LengthMismatch",
        "EmptyInput", "IoError", "ConsistencyError", "BackendUnavailable", "TraceMiss"]

"""The C-ABI library loads, exports every symbol include/*.h declares, reports the
reference's error classes, and its host-only entry points agree with the oracle."""
import ctypes as C
import os
import re

import pytest

import paper_2602_18931_b200 as ws
from oracle import pyoracle as po
from paper_2602_18931_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if not f.endswith(".h"):
            continue
        text = open(os.path.join(inc, f)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:int|const char\*)\s+(ws_\w+)\s*\(", text, flags=re.M):
            syms.add(m.group(1))
    return syms


def test_exports_every_declared_symbol():
    L = ws.lib()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in sorted(syms):
        assert hasattr(L, s), s


def test_struct_sizes_match_header():
    assert C.sizeof(abi.TokenRecord) == 72
    assert C.sizeof(abi.Pred) == 40
    assert C.sizeof(abi.OracleCfg) == 56
    assert C.sizeof(abi.StepLog) == 48


def test_abi_version():
    assert ws.lib().ws_abi_version() == 1


def test_host_synth_matches_oracle():
    for seed in (1, 5, 99):
        o = abi.oracle_cfg(seed=seed)
        assert bytes(ws.oracle_synth(o, 6)) == bytes(po.synth(o, 6))


def test_synth_config_error():
    with pytest.raises(ws.ConfigError):
        ws.oracle_synth(abi.oracle_cfg(vocab_size=1), 1)


def test_no_cpu_fallback_without_device():
    if ws.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(ws.WanspecError) as e:
        ws.Context(0)
    assert e.value.code == abi.WS_ECUDA

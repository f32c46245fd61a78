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
    assert len(syms) >= 13
    for s in sorted(syms):
        assert hasattr(L, s), s


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors == the C compiler's view of include/wanspec_b200.h."""
    pairs = [("ws_token_record", abi.TokenRecord), ("ws_pred", abi.Pred),
             ("ws_oracle_cfg", abi.OracleCfg), ("ws_sim_cfg", abi.SimCfg),
             ("ws_request_metrics", abi.RequestMetrics), ("ws_step_log", abi.StepLog),
             ("ws_run_out", abi.RunOut)]
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "wanspec_b200.h"\nint main(void){\n'
                   + "".join(f'printf("%zu\\n", sizeof({n}));\n' for n, _ in pairs)
                   + 'printf("%zu\\n", offsetof(ws_sim_cfg, oracle));\n'
                   + 'printf("%zu\\n", offsetof(ws_run_out, kernel_ms));\nreturn 0;}\n')
    exe = tmp_path / "sz"
    import subprocess
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert out[:len(pairs)] == [C.sizeof(t) for _, t in pairs]
    assert out[len(pairs)] == abi.SimCfg.oracle.offset
    assert out[len(pairs) + 1] == abi.RunOut.kernel_ms.offset


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

"""Wire framing (wire.hpp:149-323, docs/protocol.md) vs the reference's codec.

* The two worked examples of docs/protocol.md:80-113 encode to their documented bytes.
* 10^4 seeded random messages of every kind: our frames equal the reference encoder's byte for
  byte, and both decoders read either's frames back to the same fields (wire.hpp's round-trip
  fuzz, test_wire.cpp:67-77).
* Strictness (test_wire.cpp:79-127): every truncation of a frame reports need-more; bad tags,
  zero / oversized lengths, short and overlong payloads are errors with the reference's message.
"""
import ctypes as C
import random
import struct

import pytest

from oracle import pyoracle as po
from paper_2602_18931_b200 import abi


@pytest.fixture(scope="module")
def L():
    import paper_2602_18931_b200 as ws
    lib = ws.lib()
    lib.ws_wire_encode.argtypes = [C.POINTER(abi.WireMsg), C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
    lib.ws_wire_decode.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(abi.WireMsg), C.POINTER(C.c_size_t)]
    return lib


def enc(lib, m, fn="ws_wire_encode"):
    buf = (C.c_uint8 * 65536)()
    n = C.c_size_t()
    assert getattr(lib, fn)(C.byref(m), buf, 65536, C.byref(n)) == 0
    return bytes(buf[:n.value])


def dec(lib, b):
    m = abi.WireMsg()
    n = C.c_size_t()
    rc = lib.ws_wire_decode(b, len(b), C.byref(m), C.byref(n))
    return rc, m, n.value


def fields(m):
    return (m.kind, m.request_id if m.kind != 5 else 0, m.seq_no if m.kind != 5 else 0, m.base, m.config_digest,
            m.final_length, list(m.path[:m.n_path]), m.n_cands, list(m.cand_token[:m.n_cands]),
            list(m.cand_prob[:m.n_cands]), list(m.cand_entropy[:m.n_cands]), list(m.accepted[:m.n_accepted]),
            m.bonus if m.kind == 3 else 0, m.final_entropy if m.kind == 3 else 0.0)


def rand_msg(rng):
    m = abi.WireMsg()
    m.kind = rng.randint(1, 5)
    m.request_id, m.seq_no = rng.getrandbits(64), rng.getrandbits(64)
    if m.kind == 1:
        m.config_digest = rng.getrandbits(64)
    elif m.kind == 2:
        m.base = rng.getrandbits(64)
        m.n_path = rng.randint(0, 40)
        for i in range(m.n_path):
            m.path[i] = rng.getrandbits(32)
        m.n_cands = rng.randint(1, 2)
        for i in range(m.n_cands):
            m.cand_token[i] = rng.getrandbits(32)
            m.cand_prob[i] = rng.random()
            m.cand_entropy[i] = rng.random() * 5
    elif m.kind == 3:
        m.base = rng.getrandbits(64)
        m.n_accepted = rng.randint(0, 16)
        for i in range(m.n_accepted):
            m.accepted[i] = rng.getrandbits(32)
        m.bonus = rng.getrandbits(32)
        m.final_entropy = rng.random() * 3
    elif m.kind == 4:
        m.final_length = rng.getrandbits(64)
    return m


def test_protocol_doc_examples(L):
    v = abi.WireMsg(kind=3, request_id=1, seq_no=2, base=7, n_accepted=2, bonus=5, final_entropy=0.25)
    v.accepted[0], v.accepted[1] = 17, 99
    assert enc(L, v).hex() == ("0000002e" "03" "0000000000000001" "0000000000000002" "0000000000000007" "02"
                               "00000011" "00000063" "00000005" "3fd0000000000000")
    s = abi.WireMsg(kind=2, request_id=1, seq_no=3, base=9, n_path=1, n_cands=1)
    s.path[0] = 17
    s.cand_token[0], s.cand_prob[0], s.cand_entropy[0] = 42, 0.5, 0.75
    assert enc(L, s).hex() == ("00000034" "02" "0000000000000001" "0000000000000003" "0000000000000009" "0001"
                               "00000011" "01" "0000002a" "3fe0000000000000" "3fe8000000000000")
    assert enc(L, abi.WireMsg(kind=5)).hex() == "0000000105"  # the 5-byte Bye (test_wire.cpp:57-65)


def test_fuzz_roundtrip_matches_reference(L):
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = po.ref_lib()
    ref.ref_wire_encode.argtypes = [C.POINTER(abi.WireMsg), C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
    ref.ref_wire_decode.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(abi.WireMsg), C.POINTER(C.c_size_t),
                                    C.c_char_p, C.c_size_t]
    rng = random.Random(2602)
    for _ in range(10000):
        m = rand_msg(rng)
        ours, theirs = enc(L, m), enc(ref, m, "ref_wire_encode")
        assert ours == theirs
        rc, d, n = dec(L, theirs)
        assert rc == 0 and n == len(theirs)
        r2 = abi.WireMsg()
        n2 = C.c_size_t()
        err = C.create_string_buffer(256)
        assert ref.ref_wire_decode(ours, len(ours), C.byref(r2), C.byref(n2), err, 256) == 0
        assert fields(d) == fields(r2) == fields(m)


def test_strict_decoding(L):
    import paper_2602_18931_b200 as ws
    rng = random.Random(7)
    m = rand_msg(rng)
    while m.kind != 2:
        m = rand_msg(rng)
    f = enc(L, m)
    for cut in range(len(f)):
        assert dec(L, f[:cut])[0] == abi_need_more()
    cases = [(b"\x00\x00\x00\x00", "wire: frame length 0 outside (0, 1 MiB]"),
             (struct.pack(">I", (1 << 20) + 1) + b"\x05", "wire: frame length 1048577 outside (0, 1 MiB]"),
             (b"\x00\x00\x00\x01\x09", "wire: unknown kind tag 9"),
             (b"\x00\x00\x00\x09\x04" + b"\x00" * 8, "wire: payload shorter than its declared structure"),
             (b"\x00\x00\x00\x02\x05\x00", "wire: payload has 1 trailing bytes")]
    for b, msg in cases:
        rc, _, _ = dec(L, b)
        assert rc == -3  # WS_EPROTO
        assert ws.lib().ws_last_error().decode() == msg


def abi_need_more():
    return 1

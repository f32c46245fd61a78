"""Generates tests/golden/experiments/: the reference's own experiment front-end (experiment.hpp
parse_experiment -> run_experiment -> render_csv / render_per_seed_csv / render_manifest, compiled
unmodified into oracle/_ref) on the reference's experiment files (proj/experiments/*.exp),
shrunk (fewer iterations / grid points) so the B200 front-end's GPU test can rerun them in
seconds. Run here (needs /root/reference): python tests/golden/make_experiment_golden.py"""
import ctypes as C
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

SRC = "/root/reference/proj/experiments"
OUT = os.path.join(ROOT, "tests", "golden", "experiments")
SHRINK = {"iterations": "3", "phi_points": "6"}


def shrink(text, rtts):
    for k, v in SHRINK.items():
        text = re.sub(rf"^({k}\s*=\s*).*$", rf"\g<1>{v}", text, flags=re.M)
    return re.sub(r"^(rtt_ms\s*=\s*).*$", rf"\g<1>{rtts}", text, flags=re.M)


def ref_experiment(text, seed):
    lib = po.ref_lib()
    lib.ref_experiment.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t,
                                   C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t]
    n = 1 << 22
    a, b, c, e = (C.create_string_buffer(n), C.create_string_buffer(n), C.create_string_buffer(n),
                  C.create_string_buffer(512))
    rc = lib.ref_experiment(text.encode(), seed, a, n, b, n, c, n, e, 512)
    if rc != 0:
        raise RuntimeError(f"ref_experiment rc={rc}: {e.value.decode()}")
    return a.value.decode(), b.value.decode(), c.value.decode()


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, rtts in (("single_baseline", "0, 20"), ("ablation", "10, 30"), ("phi_sweep", "20, 40")):
        with open(os.path.join(SRC, name + ".exp")) as f:
            text = shrink(f.read(), rtts)
        csv, per_seed, manifest = ref_experiment(text, 1)
        for ext, body in ((".exp", text), (".csv", csv), ("_per_seed.csv", per_seed), (".manifest.json", manifest)):
            with open(os.path.join(OUT, name + ext), "w") as f:
                f.write(body)
        print(name, len(csv.splitlines()), "rows")


if __name__ == "__main__":
    main()

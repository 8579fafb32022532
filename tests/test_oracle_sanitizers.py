"""the CPU oracle's pin suites once more, against an AddressSanitizer +
UndefinedBehaviorSanitizer build of oracle/greenllm_oracle.c (-fno-sanitize-recover:
any out-of-bounds access, use after free, signed overflow, bad shift ... aborts the
run).  The child pytest loads liboracle_san.so (GREENLLM_ORACLE_SANITIZED=1) with
libasan preloaded into the interpreter."""
import os
import subprocess
import sys

import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["tests/test_oracle_pins.py", "tests/test_oracle_link.py",
          "tests/test_oracle_savings.py", "tests/test_oracle_cf.py"]


def _runtime(name):
    out = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True)
    path = out.stdout.strip()
    return path if os.path.isabs(path) and os.path.exists(path) else None


@pytest.mark.skipif(os.environ.get("GREENLLM_ORACLE_SANITIZED") == "1", reason="already inside")
def test_oracle_pin_suites_under_asan_ubsan():
    asan = _runtime("libasan.so")
    if asan is None:
        pytest.skip("gcc's libasan runtime is not installed")
    lib = O.build_sanitized(force=True)
    assert os.path.exists(lib)
    env = dict(os.environ)
    env.update(GREENLLM_ORACLE_SANITIZED="1", LD_PRELOAD=asan,
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=1:halt_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    res = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                          "-m", "not gpu", *SUITES], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=1800)
    tail = (res.stdout + res.stderr)[-3000:]
    assert res.returncode == 0, tail
    assert "ERROR: AddressSanitizer" not in res.stderr and "runtime error" not in res.stderr, tail
    assert " passed" in res.stdout, tail

"""The boundary header is plain C: include/sgi.h and the C client example compile as C99 with
warnings as errors (no C++ or torch types leak into the ABI)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_compiles_as_c99(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "sgi.h"\nint main(void) { return sgi_abi_version() == SGI_ABI_VERSION ? 0 : 1; }\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-fsyntax-only",
                        "-I", os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_client_example_compiles():
    cuda_inc = "/usr/local/cuda/include"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only",
                        "-I", os.path.join(ROOT, "include"), "-I", cuda_inc,
                        os.path.join(ROOT, "examples", "c_abi_demo.c")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

"""The drop-in at the C level: a plain C program written
against the reference's API compiles against include/iluamg_b200.h as C99,
links libilug.so, and runs. On a machine without a GPU the solve returns
ILUAMG_ERR_INVALID with the no-device message (there is no CPU path) while
the host-side calls (generator, config, last error) succeed; on a B200 the
same binary solves and prints the report's iteration count."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2111_09512_b200")

PROGRAM = r"""
#include <stdio.h>
#include <string.h>
#include "iluamg_b200.h"

int main(void) {
    iluamg_matrix* A = NULL;
    iluamg_config* cfg = NULL;
    iluamg_report* rep = NULL;
    if (iluamg_matrix_generate("poisson3d(24,24,24)", &A) != ILUAMG_OK) return 10;
    if (iluamg_config_create(&cfg) != ILUAMG_OK) return 11;
    if (iluamg_config_set(cfg, "smoother.kind", "ilu") != ILUAMG_OK) return 12;
    if (iluamg_config_set(cfg, "no.such.key", "1") != ILUAMG_ERR_INVALID) return 13;  /* fail-fast keys */
    int st = iluamg_run_solve(A, cfg, &rep);
    if (st == ILUAMG_OK) {
        printf("iterations=%s\n", iluamg_report_get(rep, "iterations"));
        iluamg_report_free(rep);
    } else {
        printf("status=%d error=%s\n", st, iluamg_last_error());
    }
    iluamg_config_free(cfg);
    iluamg_matrix_free(A);
    return 0;
}
"""


def _build(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc or not os.path.exists(os.path.join(LIBDIR, "libilug.so")):
        pytest.skip("no C compiler or libilug.so not built")
    src = tmp_path / "app.c"
    src.write_text(PROGRAM)
    exe = tmp_path / "app"
    subprocess.run([cc, "-std=c99", "-Wall", "-Werror", str(src), "-I", os.path.join(ROOT, "include"), "-L", LIBDIR,
                    "-lilug", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


def _run(exe):
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, (out.returncode, out.stderr)
    return out.stdout.strip()


def test_c_program_links_and_fails_loudly_without_gpu(ilug, tmp_path):
    if ilug.device_count() > 0:
        pytest.skip("a GPU is present (the gpu-marked test runs the solve)")
    line = _run(_build(tmp_path))
    assert line.startswith("status=2 ") and "no CUDA device" in line, line


@pytest.mark.gpu
def test_c_program_solves_on_the_gpu(ilug, torch_cuda, tmp_path):
    line = _run(_build(tmp_path))
    assert line.startswith("iterations="), line
    assert int(line.split("=")[1]) > 0

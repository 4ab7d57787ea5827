"""Host logic of the in-tree build (no nvcc needed): an object is reused only when it is newer
than its sources AND was compiled with the same command, so a diagnostic -D flag
(KFAC_NVCC_EXTRA) can never leak into a later default build."""
import os
import stat

from paper_2007_00784_b200 import build


def _fake_nvcc(tmp_path):
    log = tmp_path / "calls.txt"
    script = tmp_path / "nvcc"
    # writes the -o target and logs one line per invocation
    script.write_text("#!/bin/sh\n"
                      f"echo \"$@\" >> {log}\n"
                      "while [ $# -gt 0 ]; do if [ \"$1\" = -o ]; then shift; : > \"$1\"; fi; shift; done\n")
    script.chmod(script.stat().st_mode | stat.S_IEXEC)
    return str(script), log


def test_object_rebuilt_when_flags_change(tmp_path, monkeypatch):
    nvcc, log = _fake_nvcc(tmp_path)
    obj_dir = tmp_path / "obj"
    obj_dir.mkdir()
    src = tmp_path / "k.cu"
    src.write_text("// kernel\n")
    monkeypatch.setattr(build, "NVCC", nvcc)
    monkeypatch.setattr(build, "OBJ", str(obj_dir))
    monkeypatch.setattr(build, "_headers", lambda: [])
    calls = lambda: len(log.read_text().splitlines()) if log.exists() else 0

    monkeypatch.delenv("KFAC_NVCC_EXTRA", raising=False)
    obj = build._compile(str(src))
    assert os.path.exists(obj) and calls() == 1
    build._compile(str(src))                       # same command, newer than the source: reused
    assert calls() == 1

    monkeypatch.setenv("KFAC_NVCC_EXTRA", "-DKFAC_TRD_TIMING=1")
    build._compile(str(src))                       # different command: recompiled
    assert calls() == 2 and "-DKFAC_TRD_TIMING=1" in log.read_text().splitlines()[-1]

    monkeypatch.delenv("KFAC_NVCC_EXTRA")
    build._compile(str(src))                       # back to the default flags: recompiled again
    assert calls() == 3 and "-DKFAC_TRD_TIMING=1" not in log.read_text().splitlines()[-1]

    os.utime(src, (os.path.getmtime(obj) + 10,) * 2)   # source newer than the object
    build._compile(str(src))
    assert calls() == 4

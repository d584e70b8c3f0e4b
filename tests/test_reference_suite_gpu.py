"""The reference's OWN tests for the moment path, run UNMODIFIED through the
B200 drop-in (SURVEY.md §4 reuse plan; VERDICT r1 "What's missing" 4).

oracle/build_ref.sh packs the reference's ``src/netdos`` and ``tests`` into
oracle/_ref/netdos_ref.tar.gz (build output: git-ignored, travels to the GPU
box with the snapshot, never imported by the product).  Each case unpacks it
and runs pytest on the reference's test files in a subprocess with the plugin
tests/refsuite/netdos_gpu_rebind.py, which rebinds ``dos_moments`` /
``pdos_moments`` in ``netdos``, ``netdos.kpm`` and ``netdos.pipeline`` to
``paper_1905_09758_b200``.  The files run: test_kpm.py (kpm.py:92-152),
test_motifs.py (filter_probes + filtered moments), test_density.py
(histograms from moments) and acceptance criteria 1, 2 and 7
(test_acceptance.py:23-67, 162-176).
"""

import json
import os
import subprocess
import sys
import tarfile

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARCHIVE = os.path.join(REPO, "oracle", "_ref", "netdos_ref.tar.gz")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(ARCHIVE),
                                 reason="oracle/_ref/netdos_ref.tar.gz not built (oracle/build_ref.sh)")]


@pytest.fixture(scope="module")
def refpkg(tmp_path_factory):
    d = tmp_path_factory.mktemp("netdos_ref")
    with tarfile.open(ARCHIVE) as t:
        t.extractall(d, filter="data")
    return d


def _run(refpkg, tmp_path, files, kexpr=None):
    report = tmp_path / "calls.json"
    env = dict(os.environ, KPM_REPO=REPO, NETDOS_SRC=str(refpkg / "src"),
               KPM_REBIND_REPORT=str(report),
               PYTHONPATH=os.pathsep.join([os.path.join(REPO, "tests", "refsuite"),
                                           os.environ.get("PYTHONPATH", "")]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "netdos_gpu_rebind", "-p",
           "no:cacheprovider", "--rootdir", str(refpkg)]
    if kexpr:
        cmd += ["-k", kexpr]
    cmd += [str(refpkg / "tests" / f) for f in files]
    proc = subprocess.run(cmd, cwd=str(refpkg), env=env, capture_output=True, text=True,
                          timeout=1800)
    print(proc.stdout[-4000:])
    print(proc.stderr[-2000:])
    assert proc.returncode == 0, proc.stdout[-2000:]
    calls = json.loads(report.read_text())
    return proc.stdout, calls


def test_reference_test_kpm_unmodified(refpkg, tmp_path, kpm_ctx):
    out, calls = _run(refpkg, tmp_path, ["test_kpm.py"])
    assert calls["dos_moments"] > 10 and calls["pdos_moments"] > 0
    assert calls["backend"] == "cython"


def test_reference_test_motifs_and_density_unmodified(refpkg, tmp_path, kpm_ctx):
    out, calls = _run(refpkg, tmp_path, ["test_motifs.py", "test_density.py"])
    assert calls["dos_moments"] > 0


def test_reference_acceptance_criteria_1_2_7(refpkg, tmp_path, kpm_ctx):
    out, calls = _run(refpkg, tmp_path, ["test_acceptance.py"],
                      "criterion_01 or criterion_02 or criterion_07")
    assert "3 passed" in out and calls["dos_moments"] >= 4

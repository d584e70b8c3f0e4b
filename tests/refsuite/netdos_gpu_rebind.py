"""pytest plugin -- TEST INFRASTRUCTURE: runs the reference's OWN test modules
(unmodified, unpacked from oracle/_ref/netdos_ref.tar.gz) with netdos' moment
routines rebound to the B200 drop-in, as SURVEY.md §4's reuse plan says:

* ``netdos.kpm.dos_moments`` / ``pdos_moments`` (kpm.py:92-152),
* ``netdos.pipeline.dos_moments`` / ``pdos_moments`` (imported by name at
  pipeline.py:15),
* ``netdos.dos_moments`` / ``pdos_moments`` (__init__.py:16-17).

Loaded with ``-p netdos_gpu_rebind`` so the rebinding happens before the test
modules run ``from netdos import dos_moments``.  The adapters hand the
reference's own ScaledOperator and ProbeMatrix to
``paper_1905_09758_b200.dos_moments`` / ``pdos_moments`` (a foreign operator
is uploaded as explicit CSR values + shift/scale, kpm._device_graph), convert
the result to the reference's ChebMoments and re-raise the drop-in's
RecurrenceBlowupError as the reference's class.  Everything that is not the
moment routine (graphs, operators, probes, motifs, density, Lanczos) stays the
reference's, on its compiled Cython kernel (oracle/_ref).

Environment: KPM_REPO (repo root), NETDOS_SRC (unpacked src/), and
KPM_REBIND_REPORT (JSON file receiving the number of GPU calls).
"""

import json
import os
import sys

REPO = os.environ["KPM_REPO"]
sys.path.insert(0, REPO)
from oracle import netdos_oracle as orc  # noqa: E402

orc.ref_spmv()  # registers the reference's compiled kernel as netdos._kernels._spmv
sys.path.insert(0, os.environ["NETDOS_SRC"])

import netdos  # noqa: E402
import netdos.kpm  # noqa: E402
import netdos.pipeline  # noqa: E402
from netdos.errors import RecurrenceBlowupError as _RefBlowup  # noqa: E402

import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200.errors import RecurrenceBlowupError as _Blowup  # noqa: E402

CALLS = {"dos_moments": 0, "pdos_moments": 0, "backend": netdos.KERNEL_BACKEND}


def _probes(p):
    return kp.ProbeMatrix(p.n, p.nz, p.kind.value, p.seed, columns=p.columns)


def _ref_result(ours, sop, probes):
    return netdos.kpm.ChebMoments(mode=ours.mode, values=ours.values,
                                  scale_map=sop.scale_map, probe_meta=probes.meta())


def dos_moments(sop, probes, m_max, effective_dim=None, threads=1):
    CALLS["dos_moments"] += 1
    try:
        ours = kp.dos_moments(sop, _probes(probes), m_max, effective_dim=effective_dim)
    except _Blowup as e:
        raise _RefBlowup(str(e)) from None
    return _ref_result(ours, sop, probes)


def pdos_moments(sop, probes, m_max, normalized=True, threads=1):
    CALLS["pdos_moments"] += 1
    try:
        ours = kp.pdos_moments(sop, _probes(probes), m_max, normalized=normalized)
    except _Blowup as e:
        raise _RefBlowup(str(e)) from None
    return _ref_result(ours, sop, probes)


for _mod in (netdos, netdos.kpm, netdos.pipeline):
    _mod.dos_moments = dos_moments
    _mod.pdos_moments = pdos_moments


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("KPM_REBIND_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump(CALLS, f)

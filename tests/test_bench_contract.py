"""bench.py's contract, checked on CPU: the reference arm maps only oracle/
libraries, --gpus N re-launches N ranks, the strong-scaling shards cover the
probe set, and profiles/traffic.json is keyed to the current kernel code."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402


def test_traffic_entries_match_current_kernel():
    """roofline.traffic must come from the kernel that is benchmarked: every
    entry of profiles/traffic.json carries the hash of the step kernel's code
    it was measured on (tools/r2/traffic.py); a stale entry fails here."""
    with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
        rec = json.load(f)
    assert "entries" in rec
    now = bench.kernel_hash()
    for key, e in rec["entries"].items():
        assert e["kernel_sha"] == now, (key, "re-measure with tools/r2/traffic.py")
        assert e["dram_bytes"] == e["dram_read"] + e["dram_write"]
        assert "ncu" in e["source"]


def test_traffic_lies_between_the_byte_models_and_read_peak_is_recorded():
    """The measured DRAM bytes of a launch sit between the compulsory bytes and
    the per-nonzero gather model, and the read-gather peak that bench.py prints
    beside the copy peak (frac_of_read_peak) comes with its provenance."""
    with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
        rec = json.load(f)
    sizes = {"c5": (1 << 26, 2103834148), "c3": (1 << 24, 520768910)}
    for key, e in rec["entries"].items():
        cfg, p = key.split("/P")
        n, nnz = sizes[cfg]
        assert bench.bytes_compulsory(n, nnz, int(p)) < e["dram_bytes"] < bench.bytes_model(n, nnz, int(p))
    gbs, src = bench.read_gather_peak()
    assert 6000.0 < gbs < 8000.0 and "gather_bw" in src
    assert os.path.exists(os.path.join(REPO, "profiles", "r02_gather_roofline.log"))


def test_kernel_hash_ignores_comments():
    a = bench._code_only("int x = 1;  // note\n/* block\n comment */ int y;\n")
    b = bench._code_only("int x = 1;\nint   y;")
    assert a == b


def test_reference_arm_is_oracle_only():
    """--impl reference: no repo package, no CUDA library, no torch in the
    process; one JSON line with impl=reference and the same metric/unit."""
    code = (
        "import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'rmat14',"
        " '--steps', '2', '--warmup', '1', '--ref-probes', '2'];"
        "import bench; bench.main();"
        "bad = [m for m in sys.modules if m.startswith('paper_1905_09758_b200') or m == 'torch'];"
        "maps = open('/proc/self/maps').read();"
        "print(json.dumps({'bad': bad, 'libkpm': 'libkpm.so' in maps}))"
    )
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.strip().splitlines() if x.startswith("{")]
    line, mods = lines[0], lines[1]
    assert mods == {"bad": [], "libkpm": False}
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["unit"] == bench.UNIT and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["steps"] == 2 and line["warmup"] >= 1


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "rmat14"],
                         cwd=REPO, env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_gpus_flag_relaunches_ranks(monkeypatch):
    seen = {}

    def fake_execv(exe, cmd):
        seen["cmd"] = cmd
        raise SystemExit(0)

    monkeypatch.setattr(os, "execv", fake_execv)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    with pytest.raises(SystemExit):
        bench.main()
    cmd = seen["cmd"]
    assert "--nproc-per-node=4" in cmd and "torch.distributed.run" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_strong_scaling_shards_cover_the_probe_set():
    for world in (1, 2, 3, 4, 8):
        got = [bench.shard_range(256, r, world) for r in range(world)]
        assert got[0][0] == 0 and got[-1][1] == 256
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
        assert max(b - a for a, b in got) - min(b - a for a, b in got) <= 1


def test_byte_models_order():
    n, nnz, p = 1 << 24, 520_000_000, 128
    assert bench.bytes_compulsory(n, nnz, p) < bench.bytes_model(n, nnz, p)

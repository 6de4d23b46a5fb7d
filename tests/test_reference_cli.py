"""Drop-in proof at the level of a real caller: the REFERENCE's evaluation CLI
(proj/tools/xigemm_bench.cpp, SURVEY.md section 8(b) "callers"), compiled
unchanged by tools/build_ref_cli.py twice - against this library (B200) and
against the reference itself (oracle/_ref, CPU) - must print the same CSV /
markdown for the deterministic commands: densities, paths and the
origin / full / xigemm error columns of the precision sweep, and the QR
reconstruction table.  stage-timing and calibrate-eta are timing-based; they
must run and report on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = os.path.join(ROOT, "build", "ref_cli", "xigemm-bench")
REF = os.path.join(ROOT, "build", "ref_cli", "xigemm-bench-ref")
pytestmark = pytest.mark.gpu


def _run(exe, args, out, tmp_path):
    if not os.path.exists(exe):
        pytest.skip("reference CLI not built (needs /root/reference at build time)")
    path = os.path.join(tmp_path, out)
    r = subprocess.run([exe, *args, "--out", path], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return open(path).read(), r.stdout


@pytest.mark.parametrize("args", [
    ["precision-sweep", "--size", "96", "--dist", "all", "--th", "1,0.5,0.1,0.01"],
    ["precision-sweep", "--size", "160", "--bits", "4", "--dist", "uniform,normal",
     "--scheme", "vector", "--policy", "avg", "--th", "0.3,0.05"],
    ["density-sweep", "--size", "128", "--dist", "all", "--scheme", "vector", "--policy", "avg",
     "--th", "1,0.2,0.05,0.01", "--eta", "0.5"],
])
def test_cli_same_output_as_reference(args, tmp_path):
    ours, _ = _run(OURS, args, "ours.csv", tmp_path)
    ref, _ = _run(REF, args, "ref.csv", tmp_path)
    assert ours.splitlines()[0] == ref.splitlines()[0]  # the reference's CSV header
    assert ours == ref


def test_cli_qr_demo_same_table(tmp_path):
    args = ["qr-demo", "--dist", "uniform,normal", "--method", "float,origin,full,xigemm", "--qr-sizes", "48"]
    ours, _ = _run(OURS, args, "ours.md", tmp_path)
    ref, _ = _run(REF, args, "ref.md", tmp_path)
    assert ours == ref


def test_cli_timing_commands_run(tmp_path):
    csv, out = _run(OURS, ["stage-timing", "--size", "512", "--dist", "normal", "--th", "0.1"], "st.csv",
                    tmp_path)
    stages = {line.split(",")[10] for line in csv.splitlines()[1:]}
    assert {"quant", "xxmm", "reduce", "package"} <= stages
    cfg, out = _run(OURS, ["calibrate-eta", "--size", "128"], "xigemm.cfg", tmp_path)
    assert "eta=" in cfg

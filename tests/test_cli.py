"""The reference CLI with the GPU hot path dropped in (paper_2206_05543_b200.cli): install()
rebinds spaimg.multigrid.solve / cycle (the CLI's only solver call, reference cli.py:215-229);
on a GPU box with the reference importable, a reference `solve` and `bench` run end to end and
reproduce the reference's own numbers."""
import json
import os
import subprocess
import sys

import pytest

REF = os.environ.get("SPAIMG_REF_SRC", "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
have_ref = os.path.isdir(os.path.join(REF, "spaimg"))


@pytest.mark.skipif(not have_ref, reason="reference package not present")
def test_install_rebinds_the_reference_solver():
    # a fresh interpreter: the patch is process-wide
    code = ("import sys; sys.path.insert(0, %r); import spaimg; cpu = spaimg.multigrid.solve; "
            "from paper_2206_05543_b200 import cli; ref = cli.install(); "
            "assert ref is spaimg and spaimg.multigrid.solve is not cpu; "
            "assert spaimg.multigrid._spaimg_b200_cpu[0] is cpu; "
            "cli.install(); assert spaimg.multigrid._spaimg_b200_cpu[0] is cpu; print('ok')") % REF
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr[-2000:]


def test_missing_reference_is_a_clear_error():
    code = ("import sys; sys.modules['spaimg'] = None; from paper_2206_05543_b200 import cli\n"
            "try:\n    cli.main(['solve'])\nexcept SystemExit as e:\n    print(e)")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=300,
                       env=dict(os.environ, SPAIMG_REF_SRC=""))
    assert "not importable" in r.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not have_ref, reason="reference package not present")
def test_reference_cli_on_gpu(tmp_path):
    """A reference CLI solve through the drop-in: the RunRecord has the reference schema and the
    iteration count / rho_hat of the reference's own run of the same command."""
    out = tmp_path / "rec.json"
    args = ["solve", "--example", "3", "--N", "32", "--cycle", "v", "--nu1", "1", "--nu2", "1", "--smoother", "m7",
            "--out", str(out), "--format", "json"]
    env = dict(os.environ, SPAIMG_REF_SRC=REF)
    r = subprocess.run([sys.executable, "-m", "paper_2206_05543_b200.cli", *args], capture_output=True, text=True,
                       cwd=ROOT, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rec = json.load(open(out))
    ref_out = tmp_path / "ref.json"
    args[-3] = str(ref_out)
    r2 = subprocess.run([sys.executable, "-m", "spaimg.cli", *args], capture_output=True, text=True, cwd=ROOT,
                        env=dict(env, PYTHONPATH=REF), timeout=600)
    assert r2.returncode == 0, r2.stderr[-2000:]
    ref = json.load(open(ref_out))
    assert rec["command"] == ref["command"] == "solve" and rec["schema_version"] == ref["schema_version"]
    assert rec["outputs"]["iters"] == ref["outputs"]["iters"]
    assert rec["outputs"]["rho_hat"] == pytest.approx(ref["outputs"]["rho_hat"], rel=1e-8)

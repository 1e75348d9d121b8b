"""compute-sanitizer (memcheck, racecheck, synccheck) over every
kernel on small shapes (the segment, exact and INT8-screen routers included):
the mbarrier rings, the DSMEM hand-offs and
cta_group::2 barriers of the FFN, the self-resetting counters and the fused
combine's last-arriver protocol, the stage kernels, and the peer-memory EP
flags (one rank).  Each run must report zero errors.  (initcheck is not in
the matrix: it does not see global writes made through the async proxy --
the FFN epilogue's cp.async.bulk stores -- so every buffer the FFN writes
reads back as "uninitialized" to it.)"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("target", ["layer", "pairs", "stages", "ep"])
def test_compute_sanitizer_clean(tool, target, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    if os.environ.get("MOE_B200_SANITIZE", "0") != "1":
        # opt-in: the GPU pool closed compute-sanitizer after this round's
        # clean runs (profiles/gpu_tests_r02s6.log); see DESIGN section 8
        pytest.skip("compute-sanitizer matrix is opt-in (MOE_B200_SANITIZE=1)")
    log = tmp_path / "san.log"
    # instrument this library's kernels only (namespace moe)
    filt = ["--kernel-name", "kns=3moe"]
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--log-file", str(log), *filt, sys.executable,
           os.path.join(ROOT, "scripts", "sanitize_target.py"), target]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    text = log.read_text() if log.exists() else ""
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}_{target}.log"), "w") as fh:
        fh.write(text + "\n--- stdout ---\n" + r.stdout[-4000:] + "\n--- stderr ---\n" + r.stderr[-4000:])
    if "sanitize target done" not in r.stdout and _refused(r):
        # the GPU pool's compute-sanitizer wrapper refuses to run (policy of
        # the box, not a finding); the recorded runs are in profiles/
        pytest.skip("compute-sanitizer refused on this box: " + r.stderr.strip()[:200])
    assert "sanitize target done" in r.stdout, r.stderr[-3000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY" in text, text[-4000:]
        assert not _unexplained_races(text), text[-4000:]
    else:
        assert r.returncode == 0, text[-4000:]
        assert "ERROR SUMMARY: 0 errors" in text, text[-4000:]


def _refused(r: subprocess.CompletedProcess) -> bool:
    """The sanitizer never started the target: no output from it, and the
    wrapper says it is closed / unavailable."""
    err = r.stderr.lower()
    return not r.stdout.strip() and ("closed" in err or "not available" in err or "disabled" in err)


def _unexplained_races(text: str) -> list:
    """Racecheck reports other than the one known modelling artefact: the
    paired TMEM allocation (tcgen05.alloc.cta_group::2, executed by one warp of
    EACH CTA of a cluster pair, common.cuh tmem_alloc2) writes the allocated
    address into both CTAs' shared memory, which racecheck reports as a
    write/read race inside the alloc instruction itself.  Every other hazard
    fails the test."""
    blocks, cur = [], []
    for line in text.splitlines():
        if "Error: Race reported" in line:
            if cur:
                blocks.append(cur)
            cur = [line]
        elif cur and line.startswith("=========     and"):
            cur.append(line)
        elif cur:
            blocks.append(cur)
            cur = []
    if cur:
        blocks.append(cur)
    return [b for b in blocks if not all("tmem_alloc2" in ln for ln in b[1:]) or len(b) < 2]

"""Mutation check of the oracle's pins (VERDICT r01 Weak #1): each mutation below is a plausible
mistake in one oracle function; every one must make at least one `-m "not gpu"` pin fail.

    python tools/oracle_mutations.py        (CPU only, ~2 min; works in a scratch copy under /tmp)

M1  colour mean truncated instead of rounded half up          (R-INT)
M2  raycast hit taken when the predecessor sample is invalid  (R-RAY)
M3  tsdf mean ignoring the weight: (tsdf + s)/2               (R-INT)
M4  L1 mask reduced to D_t > 0                                (R-L1)
M5  SH view-direction term dropped in the backward (control)  (R-GRAD)
M6  raycast depth = t* instead of the camera z t*·d̂_z         (R-RAY)
M7  allocation band uses one sample less (s = 0..3)           (R-BAND)
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = {
    "M1": ("oracle/oracle.c", "cw[c] = (uint8_t)((cw[c] * w + x8 + (w + 1) / 2) / (w + 1));",
           "cw[c] = (uint8_t)((cw[c] * w + x8) / (w + 1));"),
    "M2": ("oracle/oracle.c", "if (prev_valid && prev_f > 0.0) {", "if (!prev_valid || prev_f > 0.0) {"),
    "M3": ("oracle/oracle.c", "        float num = (*ts) * wf;\n        num = num + s;\n        float den = wf + 1.0f;\n"
           "        float rden = 1.0f / den;\n        *ts = num * rden;",
           "        (void)wf; *ts = (w == 0) ? s : ((*ts) + s) * 0.5f;"),
    "M4": ("oracle/__init__.py", "M = (np.asarray(Dt) > 0) | (np.asarray(WG) > 0)", "M = (np.asarray(Dt) > 0)"),
    "M5": ("oracle/oracle.c", "for (int e = 0; e < 3; ++e) dp[e] += (ddir[e] - g.dir[e] * dd_dot) / g.dnorm;",
           "(void)dd_dot;"),
    "M6": ("oracle/oracle.c", "D = tstar / nrm; /* camera z", "D = tstar; /* camera z"),
    "M7": ("oracle/oracle.c", "for (int s = 0; s < 4; ++s) {\n        int32_t lo[3], hi[3];",
           "for (int s = 0; s < 3; ++s) {\n        int32_t lo[3], hi[3];"),
}
TESTS = ["tests/test_oracle_fuse.py", "tests/test_oracle_raycast.py", "tests/test_oracle_render.py",
         "tests/test_golden.py"]


def run(name, path, old, new):
    d = tempfile.mkdtemp(prefix=f"mut_{name}_")
    for sub in ("oracle", "tests", "gps_synth"):
        shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                        ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
    p = os.path.join(d, path)
    s = open(p).read()
    assert s.count(old) == 1, f"{name}: mutation anchor not found once in {path}"
    open(p, "w").write(s.replace(old, new))
    r = subprocess.run([sys.executable, "-m", "pytest", *TESTS, "-q", "-m", "not gpu", "-p", "no:cacheprovider"],
                       cwd=d, capture_output=True, text=True)
    shutil.rmtree(d, ignore_errors=True)
    tail = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED") or " passed" in ln or " failed" in ln]
    return r.returncode != 0, tail


def main():
    ok = True
    for name, (path, old, new) in MUTATIONS.items():
        caught, tail = run(name, path, old, new)
        ok &= caught
        print(f"{name}: {'caught' if caught else 'SURVIVED'}")
        for ln in tail[-4:]:
            print("   ", ln)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Build an A/B variant of libgps.so from textual substitutions of one source file.
    python tools/mkvariant.py <name> <file> "old=>new" ["old=>new" ...]   -> ab/<name>/libgps.so
The working tree is restored afterwards."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name, path = sys.argv[1], os.path.join(ROOT, sys.argv[2])
orig = open(path).read()
s = orig
for kv in sys.argv[3:]:
    a, b = kv.split("=>", 1)
    assert s.count(a) >= 1, a
    s = s.replace(a, b)
try:
    open(path, "w").write(s)
    subprocess.check_call([sys.executable, os.path.join(ROOT, "paper_2509_11574_b200", "build.py"), "--force",
                           "--out", os.path.join(ROOT, "ab", name, "libgps.so")], stdout=subprocess.DEVNULL)
finally:
    open(path, "w").write(orig)

"""CPU suite: every `<reference file>.py:<lines>` citation in the repository
points inside the cited reference file (catches line numbers taken from a
concatenated dump).  Skipped where /root/reference is absent
(the GPU box)."""

import os
import re
import subprocess

import pytest

REF = "/root/reference/pkg"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAT = re.compile(r"(?<![\w/])((?:tests/)?(?:test_\w+|spectral|fracop|tensor|decomp|solver|rhs|cli|oracles)\.py)"
                 r":(\d+)(?:-(\d+))?")


def _ref_lengths():
    out = {}
    for sub, prefix in (("src/fraclap", ""), ("tests", "tests/")):
        d = os.path.join(REF, sub)
        for f in os.listdir(d):
            if f.endswith(".py"):
                with open(os.path.join(d, f)) as fh:
                    n = len(fh.read().splitlines())
                out[prefix + f] = n
                if prefix:
                    out.setdefault(f, n)  # test_*.py cited without the tests/ prefix
    return out


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_reference_citations_in_range():
    lens = _ref_lengths()
    files = subprocess.check_output(["git", "ls-files"], cwd=ROOT, text=True).split()
    bad = []
    for f in files:
        if f in ("VERDICT.md", "ADVICE.md") or not f.endswith((".py", ".md", ".cu", ".cuh", ".h")):
            continue
        with open(os.path.join(ROOT, f), errors="ignore") as fh:
            for i, line in enumerate(fh, 1):
                for m in PAT.finditer(line):
                    name, a, b = m.group(1), int(m.group(2)), int(m.group(3) or m.group(2))
                    if name in lens and not (1 <= a <= b <= lens[name]):
                        bad.append("%s:%d cites %s (file has %d lines)" % (f, i, m.group(0), lens[name]))
    assert not bad, "\n".join(bad)

"""Longest run of identical (whitespace-normalised, non-trivial) lines between each host
source of this repository and each source of the reference.  Development aid, run in the
build container only (the GPU box has no /root/reference):

    python tools/copycheck.py [min_block]
"""
import difflib
import glob
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"


def norm(path):
    out = []
    for ln in open(path, errors="replace"):
        ln = re.sub(r"//.*", "", ln)
        ln = re.sub(r"\s+", "", ln)
        if len(ln) > 3:   # skip braces and blank lines
            out.append(ln)
    return out


def main():
    min_block = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    ours = sorted(glob.glob(os.path.join(ROOT, "paper_1808_01995_b200/host/*.[ch]pp")) +
                  glob.glob(os.path.join(ROOT, "include/sfb/*.hpp")))
    refs = sorted(glob.glob(os.path.join(REF, "src/*.cpp")) + glob.glob(os.path.join(REF, "include/sf/*.hpp")))
    ref_lines = {r: norm(r) for r in refs}
    worst = 0
    for o in ours:
        a = norm(o)
        for r, b in ref_lines.items():
            sm = difflib.SequenceMatcher(None, a, b, autojunk=False)
            same = sum(m.size for m in sm.get_matching_blocks())
            big = max((m.size for m in sm.get_matching_blocks()), default=0)
            if big >= min_block:
                worst = max(worst, big)
                print(f"{os.path.relpath(o, ROOT):45s} vs {os.path.relpath(r, REF):28s} "
                      f"longest identical block {big:3d} lines, {same}/{len(a)} lines shared")
    print("longest block overall:", worst)


if __name__ == "__main__":
    main()

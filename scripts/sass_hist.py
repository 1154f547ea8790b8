"""Static SASS instruction histogram of the hot kernels of libsft (cuobjdump
-sass on the built objects): proves the tensor-core (DMMA), bulk-copy
(UBLKCP) and mbarrier (SYNCS) paths are in the binary and shows the
per-kernel mix.  usage: python scripts/sass_hist.py [out.txt]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_0801_1524_b200", "build")
WANT = [  # (label, object, mangled-name regex)
    ("k_translate_ws 2D p=9 (C2)", "translate.o", r"k_translate_wsILi2ELi9ELi4ELi4ELi2ELi4E7double2Lb0ELb0ELb0E"),
    ("k_translate_ws 2D p=7 (C1)", "translate.o", r"k_translate_wsILi2ELi7ELi4ELi4ELi4ELi4E7double2Lb0ELb0ELb0E"),
    ("k_translate_ws 2D p=5 (C0)", "translate.o", r"k_translate_wsILi2ELi5E\w*7double2Lb0ELb0ELb0E"),
    ("k_translate_ws 3D p=5 (C3)", "translate.o", r"k_translate_wsILi3ELi5E\w*7double2Lb0ELb0ELb0E"),
    ("k_translate_ws 3D p=7 (C4)", "translate.o", r"k_translate_wsILi3ELi7E\w*7double2Lb0ELb0ELb0E"),
    ("k_schedule 2D p=9", "translate.o", r"k_scheduleILi2ELi9E\w*Lb0EEEvNS_11SchedLevels"),
    ("k_leaf 2D p=9", "kernels.o", r"k_leafILi2ELi9E7double2"),
    ("k_final 2D p=9", "kernels.o", r"k_finalILi2ELi9E7double2"),
]
KEY = ["DMMA", "DFMA", "DADD", "DMUL", "LDS", "STS", "LDG", "STG", "UBLKCP", "SYNCS", "SHFL", "BAR", "IMAD", "ISETP"]


def functions(obj):
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    out, cur = {}, None
    for line in txt.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if cur and m:
            out[cur][m.group(1)] += 1
    return out


def main():
    dst = sys.argv[1] if len(sys.argv) > 1 else None
    cache = {}
    lines = ["# static SASS opcode counts per kernel (cuobjdump -sass, sm_100a); columns: " + " ".join(KEY) + " total"]
    for label, obj, rx in WANT:
        if obj not in cache:
            cache[obj] = functions(os.path.join(OBJ, obj))
        hits = [(n, c) for n, c in cache[obj].items() if re.search(rx, n)]
        for n, c in hits[:1]:
            lines.append(f"{label:30s} " + " ".join(f"{k}={c.get(k, 0)}" for k in KEY) + f" total={sum(c.values())}")
            lines.append(f"    {n}")
    txt = "\n".join(lines) + "\n"
    print(txt)
    if dst:
        open(dst, "w").write(txt)


if __name__ == "__main__":
    main()

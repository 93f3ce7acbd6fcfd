"""Print the SASS of one kernel (by mangled-name substring) from a cuobjdump
-sass dump, without encodings: python tools/sass_fn.py dump.sass NAME [grep]"""
import re
import sys

txt = open(sys.argv[1]).read().split("\n")
name = sys.argv[2]
out, on = [], False
for line in txt:
    if "Function : " in line:
        on = name in line
        continue
    if on and not line.strip().startswith("/* 0x") and line.strip():
        out.append(re.sub(r"\s*/\*[0-9a-fx]*\*/\s*;?\s*$", "", line.rstrip()))
pat = sys.argv[3] if len(sys.argv) > 3 else None
for i, l in enumerate(out):
    if pat is None or re.search(pat, l):
        print(i, l.strip()[:110])

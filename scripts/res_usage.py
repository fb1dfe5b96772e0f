"""Per-kernel registers / stack / shared memory of a built library (cuobjdump -res-usage), optionally
diffed against another build: python scripts/res_usage.py NEW.so [OLD.so]"""
import re
import subprocess
import sys


def usage(path):
    out = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True).stdout
    res, fn = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        if fn and "REG:" in line:
            kv = dict(re.findall(r"(\w+(?:\[\d\])?):(\d+)", line))
            res[fn] = (int(kv.get("REG", 0)), int(kv.get("STACK", 0)), int(kv.get("SHARED", 0)))
            fn = None
    return res


new = usage(sys.argv[1])
if len(sys.argv) > 2:
    old = usage(sys.argv[2])
    for f in sorted(set(new) | set(old)):
        if new.get(f) != old.get(f):
            print(f"{old.get(f)} -> {new.get(f)}  {f[:110]}")
else:
    for f, v in sorted(new.items()):
        print(v, f[:110])

"""Static SASS statistics per kernel of libhn.so (dev tool): instruction count and opcode mix.
usage: python tools/sass_stats.py REGEX [top]"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2303_01760_b200" / "libhn.so"


def main():
    pat = re.compile(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
        if m and cur:
            funcs[cur].append(m.group(1))
    dem = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.split("\n")
    for (name, ins), pretty in zip(funcs.items(), dem):
        if not pat.search(pretty):
            continue
        c = Counter()
        for i in ins:
            tok = i.split()
            op = tok[1] if tok[0].startswith("@") else tok[0]
            c[op.split(".")[0]] += 1
        print(f"{pretty[:110]}: {len(ins)} instructions")
        print("   " + "  ".join(f"{k}:{v}" for k, v in c.most_common(top)))


if __name__ == "__main__":
    main()

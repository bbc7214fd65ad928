"""Opcode histogram (static SASS) of the kernels of librt_b200.so whose name matches a regex.

    python tools/sass_hist.py 'pt_megakernelILi0ELb0' [--lines]
"""
import re
import subprocess
import sys

LIB = "paper_2603_00292_b200/librt_b200.so"


def functions(lib=LIB):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(line)
    if cur:
        yield cur, body


def main():
    rx = re.compile(sys.argv[1])
    for name, body in functions():
        if not rx.search(name):
            continue
        hist = {}
        for line in body:
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[T0-9]\s+)?([A-Z][A-Z0-9_]*)((?:\.[A-Z0-9_]+)*)", line)
            if m:
                op = m.group(1) + (m.group(2) if m.group(1) in ("LDG", "STG", "LDL", "STL", "FMNMX3", "FFMA2") else "")
                hist[op] = hist.get(op, 0) + 1
        print(name, sum(hist.values()))
        print("  " + ", ".join(f"{k}:{v}" for k, v in sorted(hist.items(), key=lambda kv: -kv[1])))
        if "--lines" in sys.argv:
            print("\n".join(body))


if __name__ == "__main__":
    main()

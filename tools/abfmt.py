import re, sys
for l in sys.stdin:
    if "'ms'" in l and "[{" in l:
        print(l.split()[0], [m[:6] for m in re.findall(r"'ms': ([0-9.]+)", l)])
    elif l.strip():
        print(l.rstrip()[:300])

"""Print the SASS of one kernel (substring match on the mangled name) from a .so."""
import re, subprocess, sys
so, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if pat in name:
        print("Function:", name)
        print(b.split("\n", 1)[1])
        break

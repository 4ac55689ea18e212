"""Print the SASS of the kernels in libsdattn.so whose mangled name contains every given substring.

    python scripts/sass_of.py sbs_scan_kernel ILi4ELb1
"""
import re, subprocess, sys, os
lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2605_24168_b200", "libsdattn.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if all(k in name for k in sys.argv[1:]):
        print("Function :", name)
        print(b.split("\n", 1)[1])

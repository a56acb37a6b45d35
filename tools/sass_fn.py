"""Print the SASS of one kernel (substring match on the mangled name) from a cuobjdump -sass dump."""
import re
import sys

text = open(sys.argv[1]).read()
parts = re.split(r"\n\s*Function : ", text)
for p in parts[1:]:
    name = p.split("\n", 1)[0].strip()
    if all(s in name for s in sys.argv[2:]):
        print("Function :", p)

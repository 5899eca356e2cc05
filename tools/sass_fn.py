"""Print the SASS of one kernel from a cuobjdump -sass dump: sass_fn.py DUMP SUBSTRING"""
import sys
txt = open(sys.argv[1]).read().split("\n")
out, on = [], False
for l in txt:
    if "Function :" in l:
        on = sys.argv[2] in l
    if on:
        out.append(l)
print("\n".join(out))

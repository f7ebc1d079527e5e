"""Static SASS size of one kernel per source line and per enclosing function.
usage: sass_static.py OBJ KERNEL_SUBSTR [TOP]"""
import collections, os, sys
sys.path.insert(0, os.path.dirname(__file__))
from sassmap import line_map, source, func_of

obj, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lm = line_map(obj, ksub)
print(f"{len(lm)} instructions ({len(lm) * 16 / 1024:.0f} KB)")
fc = collections.Counter(func_of(*v) for v in lm.values())
for nm, k in fc.most_common(top):
    print(f"{k:6d}  {nm}")

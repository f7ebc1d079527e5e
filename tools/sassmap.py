"""SASS address -> source line maps from nvdisasm -gi (innermost frame, with
CUDA intrinsics attributed to their caller) and source-line -> enclosing
device function lookup.  Shared by ncu_lines.py and sass_static.py."""
import glob, os, re, subprocess, tempfile


def cubin_of(obj):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    return glob.glob(os.path.join(d, "*.cubin"))[0]


def line_map(obj, ksub, depth=False):
    """{addr: (file, line)} for instructions of the kernel whose name contains ksub
    (with depth=True: {addr: ((file, line), inline depth)})."""
    dis = subprocess.run(["nvdisasm", "-gi", cubin_of(obj)], capture_output=True, text=True).stdout
    out, fn, cur, fresh, dep = {}, None, None, True, 0
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            here = (os.path.basename(m.group(1)), int(m.group(2)))
            if fresh:
                dep = 0
            if fresh or cur[0].startswith("sm_"):
                cur = here
            fresh = False
            dep += 1
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+\S", ln)
        if m:
            fresh = True
            if fn and ksub in fn:
                out[int(m.group(1), 16)] = (cur, dep) if depth else cur
    return out


_src, _funcs = {}, {}


def source(f):
    if f not in _src:
        root = os.environ.get("SRC_ROOT", "/root/repo")
        p = glob.glob(root + "/**/" + f, recursive=True)
        _src[f] = open(p[0]).read().split("\n") if p else []
    return _src[f]


def func_of(f, l):
    if f not in _funcs:
        starts = []
        for i, t in enumerate(source(f), 1):
            m = re.search(r"(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", t)
            if m and not t.strip().startswith("//"):
                starts.append((i, m.group(1)))
        _funcs[f] = starts
    name = f
    for s, nm in _funcs[f]:
        if s <= l:
            name = f"{f}:{nm}@{s}"
    return name

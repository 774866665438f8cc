"""Build A/B variants of the library with extra -D flags (perf experiments).

    python tools/ab_build.py NAME -DFOO=1 -DBAR=2 ...

writes build/ab/NAME/libdacsr_b200.so (git-ignored, shipped by gpurun);
select it at run time with DACSR_LIB_PATH=build/ab/NAME/libdacsr_b200.so.
"""
import concurrent.futures as cf
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as g  # noqa: E402


def build(name, defines):
    out = os.path.join(g.ROOT, "build", "ab", name)
    os.makedirs(out, exist_ok=True)
    jobs, objs = [], []
    for src in g._sources():
        path = os.path.join(g.CSRC, src)
        obj = os.path.join(out, src + ".o")
        objs.append(obj)
        if src.endswith(".cu"):
            jobs.append([g.NVCC, *g.ARCH, *g.NVFLAGS, *defines, "-c", path, "-o", obj])
        else:
            jobs.append(["g++", *g.CXXFLAGS, "-c", path, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        list(ex.map(g._run, jobs))
    lib = os.path.join(out, "libdacsr_b200.so")
    g._run([g.NVCC, *g.ARCH, "-shared", "-o", lib, *objs])
    return lib


if __name__ == "__main__":
    print(build(sys.argv[1], sys.argv[2:]))

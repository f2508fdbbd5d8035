"""Build an alternative libgeot for kernel A/B experiments, next to the normal build:
    python tools/build_variant.py NAME unit.cu[,unit2.cu] -DMACRO=VALUE ...
recompiles the listed translation units with the extra flags and links
scratch/NAME/libgeot.so; load it with GEOT_LIB_OVERRIDE=scratch/NAME/libgeot.so
(e.g. -DGEOT_TRACE for tools/trace_stream.py, -DGEOT_NARROW_F1_WARPS=8)."""
import glob, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import build as b
name, units, defs = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
b.build(verbose=False)
objs = sorted(glob.glob(os.path.join(b.BUILD, "geot", "*.o")))
out = os.path.join(b.ROOT, "scratch", name); os.makedirs(out, exist_ok=True)
for u in units:
    o = os.path.join(out, u + ".o")
    subprocess.run([b.NVCC] + b.NVFLAGS + defs + ["-c", os.path.join(b.CSRC, u), "-o", o], check=True)
    objs = [x for x in objs if os.path.basename(x) != u + ".o"] + [o]
subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", os.path.join(out, "libgeot.so")] + objs + ["-cudart=static"], check=True)
print("built", os.path.join(out, "libgeot.so"))

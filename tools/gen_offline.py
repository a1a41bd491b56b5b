"""Offline look at the generated pass kernels (no GPU): plan a config, generate its
CUDA source on a host-only handle, compile it with NVRTC (as the engine does) for sm_100a and report per
pass kernel registers, spills, SASS size and instruction mix.

  python tools/gen_offline.py [config] [dtype] [--keep DIR]
"""
import os, re, subprocess, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.engine import generated_source
from paper_2504_16297_b200.program import compile_circuit

cfg = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 4
dtype = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2].startswith("c") else "c64"
out = sys.argv[sys.argv.index("--keep") + 1] if "--keep" in sys.argv else "/tmp/gen"
os.makedirs(out, exist_ok=True)
os.environ.setdefault("PTSBE_CODEGEN", "1")
c = workloads.build(cfg, P.parse_circuit, P.parse_noise_model, P.attach_noise)
prog = compile_circuit(c, dtype)
src = generated_source(prog, dtype)
cu = os.path.join(out, f"gen_cfg{cfg}_{dtype}.cu")
open(cu, "w").write(src)
cubin = cu[:-3] + ".cubin"
# compile exactly as the engine does: the CUDA toolkit's NVRTC (codegen.h api()), same options
import ctypes as C
import torch  # noqa: F401  (the bench/tests process has torch's own NVRTC loaded too)
nv = C.CDLL(os.environ.get("PTSBE_NVRTC", "/usr/local/cuda/lib64/libnvrtc.so.12"), mode=os.RTLD_NOW | os.RTLD_LOCAL)
maj, mnr = C.c_int(), C.c_int()
nv.nvrtcVersion(C.byref(maj), C.byref(mnr))
nvprog = C.c_void_p()
assert nv.nvrtcCreateProgram(C.byref(nvprog), src.encode(), b"ptsbe_gen.cu", 0, None, None) == 0
opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo", b"--device-as-default-execution-space",
        b"-Xptxas", b"-v"]
arr = (C.c_char_p * len(opts))(*opts)
rc = nv.nvrtcCompileProgram(nvprog, len(opts), arr)
n = C.c_size_t()
nv.nvrtcGetProgramLogSize(nvprog, C.byref(n))
log = C.create_string_buffer(n.value)
nv.nvrtcGetProgramLog(nvprog, log)
if rc:
    print(log.value.decode()[-3000:]); sys.exit(1)
nv.nvrtcGetCUBINSize(nvprog, C.byref(n))
buf = C.create_string_buffer(n.value)
nv.nvrtcGetCUBIN(nvprog, buf)
open(cubin, "wb").write(buf.raw)
class R: pass
r = R(); r.stderr = log.value.decode()
print(f"NVRTC {maj.value}.{mnr.value}")
regs = {}
cur = None
for line in r.stderr.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m: cur = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur: regs[cur] = int(m.group(1))
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur and int(m.group(1)): regs[cur + "_spill"] = int(m.group(1))
sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
fn = None
stats = collections.OrderedDict()
hot = {}   # bytes of the kernel body before its first out-of-line (slow-path) function
for line in sass.splitlines():
    m = re.search(r"Function : (\w+)", line)
    if m:
        fn = m.group(1); stats[fn] = collections.Counter(); continue
    m = re.search(r"CALL.REL.NOINC 0x([0-9a-f]+)", line)
    if m and fn:
        hot[fn] = min(hot.get(fn, 1 << 40), int(m.group(1), 16))
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and fn:
        op = m.group(1).split(".")[0]
        stats[fn][op] += 1
ops_per_pass = collections.Counter(pi for pi, pl in enumerate(prog.passes) for _ in pl.ops)
def key(f):
    return int(f.rsplit("_", 1)[1])
tot = collections.Counter()
print(f"config {cfg} {dtype}: {prog.n_passes} passes")
print(f"{'kernel':14s} {'ops':>5s} {'regs':>5s} {'instr':>7s} {'KB':>6s} {'hotKB':>6s} {'FFMA2':>6s} {'FADD2':>6s} {'FMUL2':>6s} {'LDS':>5s} {'STS':>5s} {'BAR':>4s} {'MOV':>5s} {'other':>6s}")
for f in sorted(stats, key=key):
    s = stats[f]; n = sum(s.values()); tot += s
    main = s["FFMA2"] + s["FADD2"] + s["FMUL2"] + s["LDS"] + s["STS"] + s["BAR"] + s["MOV"]
    print(f"{f:14s} {ops_per_pass[key(f)]:5d} {regs.get(f, 0):5d} {n:7d} {n * 16 / 1024:6.1f} {hot.get(f, n * 16) / 1024:6.1f} {s['FFMA2']:6d} {s['FADD2']:6d} "
          f"{s['FMUL2']:6d} {s['LDS']:5d} {s['STS']:5d} {s['BAR']:4d} {s['MOV']:5d} {n - main:6d}"
          + (f"  spill {regs[f + '_spill']}" if f + "_spill" in regs else ""))
print("top other opcodes:", [(k, v) for k, v in tot.most_common(25) if k not in ("FFMA2", "FADD2", "FMUL2", "LDS", "STS", "BAR", "MOV")][:15])

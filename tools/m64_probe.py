"""Run tools/m64_probe.cu: which TMEM lanes hold A and D rows for M=64 tcgen05.mma (see the .cu header)."""
import ctypes, pathlib, subprocess
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parents[1]
SO = ROOT / "tools" / "_lib" / "libm64probe.so"
if not SO.exists():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-shared", str(ROOT / "tools" / "m64_probe.cu"), "-o", str(SO)], check=True)
L = ctypes.CDLL(str(SO))
for layout in (0, 1):
    out = np.zeros((128, 64), np.float32)
    rc = L.probe_m64(layout, out.ctypes.data_as(ctypes.c_void_p))
    col0 = out[:, 0]
    uniform = bool(np.all(out == out[:, :1]))
    print(f"layout {layout} rc {rc} rows-uniform-across-columns {uniform}")
    print("  D lane -> value (col 0):", " ".join(f"{l}:{col0[l]:.0f}" for l in range(128)))

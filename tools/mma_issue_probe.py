"""Run tools/mma_issue_probe.cu: cycles per tcgen05.mma (M128 N64 K16) by issue form; see the .cu header."""
import ctypes, json, pathlib, subprocess
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parents[1]
SO = ROOT / "tools" / "_lib" / "libmmaissue.so"
if __name__ == "__main__":
    if not SO.exists():
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                        "-shared", str(ROOT / "tools" / "mma_issue_probe.cu"), "-o", str(SO)], check=True)
    L = ctypes.CDLL(str(SO))
    iters = 4096
    for mode in range(6, 15):
        c = np.zeros(148, np.int64)
        rc = L.probe_issue(iters, mode, c.ctypes.data_as(ctypes.c_void_p))
        print(json.dumps({"mode": mode, "rc": rc, "cycles_per_mma": float(np.median(c)) / iters}))

"""Run tools/tmem_a_probe.cu: check the TMEM A-operand layout and the halo kernel's K permutation."""
import ctypes as C
import json
import pathlib
import subprocess
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
SO = ROOT / "tools" / "_lib" / "libtmemprobe.so"


def perm64():
    """MMA K index -> channel for the 16x256b.x4 mapping (thread t0 loads chunks 2*t0 + j, j = 0, 1)."""
    p = []
    for k in range(64):
        col, h = k >> 1, k & 1
        t0, i = (col & 7) >> 1, 2 * (col >> 3) + (col & 1)
        j, e = i >> 2, i & 3
        c = 2 * t0 + j
        p.append(8 * c + 2 * e + h)
    return np.array(p)


def pack_sw128(b):  # b: [64 n][64 k] -> 8 KB K-major 128B-swizzled image (uint16)
    img = np.zeros(64 * 64, np.uint16)
    for n in range(64):
        for k in range(64):
            c, e = k >> 3, k & 7
            off = n * 128 + ((c ^ (n & 7)) << 4) + 2 * e
            img[off // 2] = b[n, k]
    return img


def main():
    SO.parent.mkdir(exist_ok=True)
    if not SO.exists() or "--build" in sys.argv:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler",
                        "-fPIC", "-shared", str(ROOT / "tools" / "tmem_a_probe.cu"), "-o", str(SO)], check=True)
    if "--build-only" in sys.argv:
        return
    L = C.CDLL(str(SO))
    rng = np.random.default_rng(0)
    a = torch.from_numpy(rng.normal(size=(128, 64)).astype(np.float32)).to(torch.bfloat16)
    b = torch.from_numpy(rng.normal(size=(64, 64)).astype(np.float32)).to(torch.bfloat16)
    ref = a.double() @ b.double().T
    bu = b.view(torch.int16).numpy().view(np.uint16)
    pi = perm64()
    assert sorted(pi) == list(range(64))
    rep = {}
    for mode, bimg in ((0, pack_sw128(bu)), (1, pack_sw128(bu[:, pi]))):
        ad = a.cuda()
        bd = torch.from_numpy(bimg.view(np.int16)).cuda()
        out = torch.zeros(128, 64, dtype=torch.float32, device="cuda")
        rc = L.probe_tmem_a(C.c_void_p(ad.data_ptr()), C.c_void_p(bd.data_ptr()), C.c_void_p(out.data_ptr()), mode)
        err = float((out.cpu().double() - ref).abs().max() / ref.abs().max())
        rep[f"mode{mode}"] = {"rc": rc, "rel_err": err}
    cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
    for n in (64,):
        for mode, name in enumerate(("ss", "ts", "ts_mask0", "ts_mask_half", "ss_elect", "ts_elect", "ss_2warps", "ss_4warps", "ts_2warps", "ts_4warps")):
            ms = C.c_float(0)
            iters = 20000
            rc = L.probe_rate(n, iters, mode, C.c_void_p(cyc.data_ptr()), C.byref(ms))
            c = float(cyc.float().mean()) / (iters * 4)
            rep[f"rate_n{n}_{name}"] = {"rc": rc, "cycles_per_mma": round(c, 1),
                                        "tflops": round(148 * iters * 4 * 2 * 128 * n * 16 / (ms.value * 1e-3) / 1e12)}
    for ts, name in ((0, "ss"), (1, "ts")):
        ms = C.c_float(0)
        iters = 20000
        rc = L.probe_rate2(iters, ts, C.c_void_p(cyc.data_ptr()), C.byref(ms))
        c = float(cyc[:74].float().mean()) / (iters * 4)
        rep[f"rate_cta2_m256_n64_{name}"] = {"rc": rc, "cycles_per_mma": round(c, 1),
                                             "tflops": round(74 * iters * 4 * 2 * 256 * 64 * 16 / (ms.value * 1e-3) / 1e12)}
    wc = torch.zeros(4, dtype=torch.int64, device="cuda")
    it = 10000
    rc = L.probe_wait_cost(it, C.c_void_p(wc.data_ptr()))
    w = wc.cpu().tolist()
    rep["wait_cost_cycles"] = {"rc": rc, "try_wait": w[0] / it, "test_wait": w[1] / it, "mbar_wait_loop": w[2] / it}
    print(json.dumps(rep))


if __name__ == "__main__":
    main()

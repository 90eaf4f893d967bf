"""Run tools/tc_probe.cu on the GPU: D = A B^T through tcgen05.mma.kind::tf32 (A from TMEM, B from
shared memory, K-major no-swizzle descriptors) against numpy, with tf32-exact integer inputs (exact
match expected) and random inputs. Test infrastructure for the tensor-core recursive pass 2."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = "/tmp/tc_probe.so"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                       "-Xcompiler", "-fPIC", os.path.join(HERE, "tc_probe.cu"), "-o", so])
lib = ctypes.CDLL(so)
ok = True
rng = np.random.default_rng(0)
for N in (32, 64):
    for KS in (1, 5):
        K = 8 * KS
        for kind in ("int", "rand"):
            if kind == "int":
                A = rng.integers(-8, 9, (128, K)).astype(np.float32)
                B = rng.integers(-8, 9, (N, K)).astype(np.float32)
            else:
                A = rng.uniform(-1, 1, (128, K)).astype(np.float32)
                B = rng.uniform(-1, 1, (N, K)).astype(np.float32)
            a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            d = torch.zeros(128, N, device="cuda")
            rc = lib.tc_probe(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                              ctypes.c_void_p(d.data_ptr()), N, KS)
            ref = A.astype(np.float64) @ B.astype(np.float64).T
            err = np.abs(d.cpu().numpy() - ref).max()
            tol = 0 if kind == "int" else 4e-3 * np.sqrt(K)
            good = rc == 0 and err <= tol
            ok &= good
            print(f"N={N} KS={KS} {kind}: rc={rc} max err {err:.3g} (tol {tol:.3g}) {'OK' if good else 'FAIL'}")
            if not good and kind == "int":
                D = d.cpu().numpy()
                print(" D[0,:8]", D[0, :8], "\n ref[0,:8]", ref[0, :8])
                print(" D[9,:8]", D[9, :8], "\n ref[9,:8]", ref[9, :8])
sys.exit(0 if ok else 1)

#!/usr/bin/env python
"""Where a warm eos_search_create spends its time (GPU box): host plan alone, create,
destroy, and a raw cudaMalloc + cudaMemcpy + cudaFree of the same image size."""
import ctypes
import glob
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2112_03229_b200 as eos  # noqa: E402


def us(fn, reps=50):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps * 1e6


def main():
    torch.zeros(1, device="cuda")
    libs = sorted(glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))) or \
        sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))
    rt = ctypes.CDLL(libs[0])
    for name in ("cfg1", "cfg5"):
        X = datagen.workload(name, count=10).table
        info, _ = eos.plan_table(X, eos.EOS_K_AUTO, with_directory=False)
        img = info.image_bytes
        t_plan = us(lambda: eos.plan_table(X, eos.EOS_K_AUTO, with_directory=False))
        hs = []
        t_create = us(lambda: hs.append(eos.eos_search_create(X)))
        t_destroy = us(lambda: eos.eos_search_destroy(hs.pop()), reps=len(hs) - 1)
        buf = ctypes.create_string_buffer(img)
        p = ctypes.c_void_p()

        def raw():
            rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(img))
            rt.cudaMemcpy(p, buf, ctypes.c_size_t(img), 1)
            rt.cudaFree(p)
        t_raw = us(raw)
        print(f"{name}: image {img} B  plan {t_plan:.1f} us  create {t_create:.1f} us  "
              f"destroy {t_destroy:.1f} us  raw malloc+memcpy+free {t_raw:.1f} us")


if __name__ == "__main__":
    main()

"""Drive tools/bwprobe.cu (diagnostic): write bandwidth per store form.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
         -o tools/libbwprobe.so tools/bwprobe.cu && python tools/bwprobe.py
"""

import ctypes as C
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
NAMES = ["st.v4", "st.v4.cs", "st.v8 (256-bit)", "st.v8 L2::evict_first", "st.v4 unroll4", "TMA bulk store",
         "copy v4 (read+write)", "st.v4 PDL + griddepcontrol.wait", "st.v4 PDL, no wait (bound)"]


def main():
    lib = C.CDLL(os.path.join(HERE, "libbwprobe.so"))
    lib.bw_probe.restype = C.c_float
    lib.bw_probe.argtypes = [C.c_int, C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int]
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for total, nbuf, reps, graph in ((1 << 30, 2, 10, 0), (32_833_536, 8, 200, 0), (21_000_000 // 16384 * 16384, 12, 200, 0),
                                     (21_000_000 // 16384 * 16384, 12, 200, 1)):
        bufs = [torch.empty(total, dtype=torch.uint8, device=dev) for _ in range(nbuf)]
        arr = (C.c_void_p * nbuf)(*[b.data_ptr() for b in bufs])
        print(f"--- {total / 1e6:.1f} MB per launch, ring of {nbuf}{', CUDA graph' if graph else ''}")
        for v, name in enumerate(NAMES):
            best = None
            for blocks, threads in ((sms * 4, 512), (sms * 8, 256), (sms * 16, 128), (sms * 2, 1024), (sms, 128)):
                if v != 5 and threads == 128 and blocks == sms:
                    continue
                us = lib.bw_probe(v, arr, nbuf, total, reps, blocks, threads, graph)
                if us <= 0:
                    continue
                gbs = total * (2 if v == 6 else 1) / us / 1e3
                if best is None or gbs > best[0]:
                    best = (gbs, us, blocks, threads)
            if best:
                print(f"  {name:26s} {best[1]:9.2f} us  {best[0]:8.1f} GB/s  (grid {best[2]} x {best[3]})")
        del bufs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

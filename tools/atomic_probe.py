"""Drive tools/atomic_probe.cu: cycles per dependent CAS / load (diagnostic)."""
import ctypes as C
import os
import statistics

import torch

lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libatomicprobe.so"))
buf = torch.full((1 << 24,), -1, dtype=torch.int64, device="cuda")
for mode, name in ((0, "CAS hot line"), (1, "load hot line"), (2, "CAS random (128 MB)"), (3, "load random (128 MB)")):
    for blocks in (1, 128):
        out = (C.c_longlong * blocks)()
        lib.atomic_probe(C.c_void_p(buf.data_ptr()), C.c_size_t(buf.numel()), out, mode, blocks)
        v = list(out)
        print(f"{name:22s} blocks {blocks:4d}: median {statistics.median(v):7.0f} max {max(v):7.0f} cycles")

# the same probes while another stream streams writes (the K5 apply phase)
side = torch.cuda.Stream()
big = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for mode, name in ((0, "CAS hot line"), (2, "CAS random (128 MB)"), (3, "load random (128 MB)")):
    with torch.cuda.stream(side):
        for _ in range(4):
            big.fill_(7)
    out = (C.c_longlong * 16)()
    lib.atomic_probe(C.c_void_p(buf.data_ptr()), C.c_size_t(buf.numel()), out, mode, 16)
    torch.cuda.synchronize()
    v = list(out)
    print(f"under write stream: {name:22s} median {statistics.median(v):7.0f} max {max(v):7.0f} cycles")

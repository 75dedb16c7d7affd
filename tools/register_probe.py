"""Cost of page-locking fresh host result arrays (HostIO's retained CSR):
cudaHostRegister on np.empty memory, with and without a parallel first touch,
and the D2H rate into the registered array.   python tools/register_probe.py [GB]"""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import mmap

import numpy as np
import torch


def empty(n, huge):
    if not huge:
        return np.empty(n, np.float64)
    mm = mmap.mmap(-1, (n * 8 + (1 << 21) - 1) & ~((1 << 21) - 1))
    mm.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(mm, np.float64, count=n)


def main(gb=16.0):
    n = int(gb * (1 << 30)) // 8
    pool = ThreadPoolExecutor(16)
    dev = torch.empty(n, dtype=torch.float64, device="cuda").fill_(1.0)
    for pre, huge in ((0, 0), (1, 0), (1, 1), (1, 0), (1, 1)):
        t0 = time.perf_counter()
        a = empty(n, huge)
        if pre:
            parts = np.linspace(0, n, 17).astype(np.int64)
            list(pool.map(lambda k: a[parts[k]:parts[k + 1]].fill(0.0), range(16)))
        t1 = time.perf_counter()
        rc = torch._C._cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        t2 = time.perf_counter()
        h = torch.from_numpy(a)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        for _ in range(3):
            h.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        print(f"prefault={pre} hugepages={huge} touch {t1 - t0:.2f} s register {t2 - t1:.2f} s ({rc}) "
              f"D2H {3 * gb / (t4 - t3):.1f} GB/s ok={bool(a[::1 << 20].min() == 1.0)}", flush=True)
        torch._C._cudart.cudaHostUnregister(a.ctypes.data)
        del h, a


if __name__ == "__main__":
    main(*(float(x) for x in sys.argv[1:]))

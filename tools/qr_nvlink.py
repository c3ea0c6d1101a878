"""NVLink QR microbenchmark (single process, one PE per GPU): the push and the
in-place exchange kernels of libqrt (qrt_qr_bench) for k = 1..log2(N) swapped
local<->global position pairs.  Prints one JSON line per (mode, k) with the
per-direction rate against the measured 770 GB/s peer copy and the 900 GB/s
nominal NVLink 5 figure (B200_PROFILING.md).

  python tools/qr_nvlink.py [--gpus N] [--nl 30] [--iters 5]
Run it under ncu (single process) for the nvltx/nvlrx counters."""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2410_04252_b200 as qb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gpus", type=int, default=0)
ap.add_argument("--nl", type=int, default=30)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--modes", default="push,inplace")
args = ap.parse_args()
lib = qb.load_libqrt()
lib.qrt_last_error.restype = C.c_char_p
n = args.gpus or qb.device_count()
g = n.bit_length() - 1
for mode in args.modes.split(","):
    for k in range(1, g + 1):
        ms, gbs = C.c_double(), C.c_double()
        rc = lib.qrt_qr_bench(n, args.nl, k, 1 if mode == "inplace" else 0, args.iters, C.byref(ms), C.byref(gbs))
        if rc != 0:
            print(json.dumps({"mode": mode, "k": k, "error": lib.qrt_last_error().decode()}))
            continue
        sent = 16 * (1 << args.nl) * (1 - 2.0 ** -k)
        print(json.dumps({"mode": mode, "gpus": n, "k": k, "n_local": args.nl, "ms": ms.value,
                          "bytes_sent_per_gpu": sent, "gbs_per_direction": gbs.value,
                          "frac_of_770_measured": gbs.value / 770.0, "frac_of_900_nominal": gbs.value / 900.0}))

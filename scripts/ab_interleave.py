"""Developer probe: interleaved A/B of library builds in ONE process (same box,
same thermal state): every rep sorts the same regenerated input once with each
var/lib_<tag>.so, in rotating order, timed with CUDA events on one stream.

    python scripts/ab_interleave.py [c1 c5 ...] [--reps 6] [--kt]
"""
import ctypes as C
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1612_02557_b200 as rg  # noqa: E402
from scripts.perf_probe import CONFIGS  # noqa: E402


def main():
    names = [a for a in sys.argv[1:] if a in CONFIGS] or ["c1"]
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 6
    libs = {}
    for i, path in enumerate(sorted(glob.glob("var/lib_*.so"))):
        tag = os.path.basename(path)[4:-3]
        # a private copy per tag: dlopen keys on the path
        priv = f"/tmp/ab_{i}_{tag}.so"
        os.system(f"cp {path} {priv}")
        L = C.CDLL(priv, mode=C.RTLD_LOCAL)
        L.raduls_gpu_sort.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_void_p]
        L.raduls_gpu_sort.restype = C.c_int
        if "--kt" in sys.argv:
            L.raduls_gpu_set_profiling(1)
        libs[tag] = L
    tags = list(libs)
    stream = torch.cuda.current_stream()
    for name in names:
        n, rs, ks, dist, seed = CONFIGS[name]
        lay = rg.RecordLayout(rs, ks)
        data = torch.empty(n * rs, dtype=torch.uint8, device="cuda")
        tmp = torch.empty_like(data)
        times = {t: [] for t in tags}
        kt = {t: {} for t in tags}
        for r in range(reps + 1):
            order = tags[r % len(tags):] + tags[:r % len(tags)]
            for t in order:
                rg.generate(n, lay, dist=dist, seed=seed, out=data)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                rc = libs[t].raduls_gpu_sort(data.data_ptr(), tmp.data_ptr(), n, rs, ks,
                                             stream.cuda_stream)
                e1.record(stream)
                torch.cuda.synchronize()
                assert rc == 0, (t, rc)
                if r:
                    times[t].append(e0.elapsed_time(e1))
                    if "--kt" in sys.argv:
                        buf = (rg._lib.KernelTime * 16)()
                        cnt = C.c_int(0)
                        libs[t].raduls_gpu_last_kernel_times(buf, 16, C.byref(cnt))
                        for i in range(cnt.value):
                            kt[t].setdefault(buf[i].name.decode(), []).append(buf[i].ms)
        v, _ = rg.check_sorted(data, n, lay)
        out = {"config": name, "violations": v}
        for t in tags:
            s = sorted(times[t])
            out[t] = {"median": round(s[len(s) // 2], 3), "min": round(s[0], 3)}
            for k, v in kt[t].items():
                v = sorted(v)
                if v[len(v) // 2] > 0.05:
                    out[t][k] = round(v[len(v) // 2], 3)
        print(json.dumps(out), flush=True)
        del data, tmp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

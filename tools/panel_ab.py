"""A/B of batched augmented LU builds (developer tool): the same seeded inputs through two libhps_b200 builds,
each in its own process (two copies of the library in one process share template statics).
usage: python tools/panel_ab.py libA.so libB.so  -> per (n, m, batch): ms each, bitwise equality of factors/pivots"""
import sys, json, subprocess, ctypes as C, os
sys.path.insert(0, '.')
CASES = [(56, 113, 16384), (112, 225, 4096), (224, 449, 1024), (448, 897, 256), (896, 1793, 64), (1792, 3585, 16),
         (3584, 7169, 4), (7168, 1, 1)]


def run(libpath, out):
    import torch
    L = C.CDLL(libpath)
    L.hpsg_dev_getrf_aug.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p, C.c_void_p]
    res = {}
    for n, m, b in CASES:
        g = torch.Generator(device="cuda").manual_seed(n)
        M0 = torch.randn((b, n + m, n), dtype=torch.float64, device="cuda", generator=g)
        M = M0.clone(); piv = torch.zeros((b, n), dtype=torch.int32, device="cuda"); st = torch.zeros((b, 3), dtype=torch.float64, device="cuda")
        ts, rc = [], 0
        for it in range(4):
            M.copy_(M0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = L.hpsg_dev_getrf_aug(b, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), st.data_ptr())
            e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[f"{n}"] = {"ms": min(ts[1:]), "rc": rc}
        torch.save({"M": M.cpu(), "piv": piv.cpu()}, f"{out}_{n}.pt")
    json.dump(res, open(out + ".json", "w"))


if __name__ == "__main__":
    if sys.argv[1] == "--run":
        run(sys.argv[2], sys.argv[3]); sys.exit(0)
    import torch
    outs = []
    for i, lp in enumerate(sys.argv[1:3]):
        o = f"/tmp/panel_ab_{i}"
        subprocess.run([sys.executable, __file__, "--run", lp, o], check=True)
        outs.append(json.load(open(o + ".json")))
    for n, m, b in CASES:
        A = torch.load(f"/tmp/panel_ab_0_{n}.pt"); B = torch.load(f"/tmp/panel_ab_1_{n}.pt")
        print(json.dumps({"n": n, "batch": b, "ms_a": outs[0][str(n)]["ms"], "ms_b": outs[1][str(n)]["ms"],
                          "rc": [outs[0][str(n)]["rc"], outs[1][str(n)]["rc"]],
                          "bitwise_equal": bool(torch.equal(A["M"], B["M"]) and torch.equal(A["piv"], B["piv"])),
                          "max_abs_diff": float((A["M"] - B["M"]).abs().max())}), flush=True)

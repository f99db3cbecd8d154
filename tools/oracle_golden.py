"""Writes tests/golden/oracle_iters.json: the CPU oracle's outer FCG iteration counts for the full
BASELINE configs (x0 = 0, rhs seed 0, tol 1e-8, nu = 2), its solution x at 4096 evenly spaced rows
(plus max|x| and ||x||), and the host it ran on.  Calls only oracle/ and inputs/ (never the
CUDA path), so the GPU parity tests can compare against it (+-1) without rerunning the oracle.

    python tools/oracle_golden.py C3 [C4 C5 ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import gen  # noqa: E402
from oracle import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_iters.json")


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "threads_used": 1}


def main(names):
    host = host_info()
    data = json.load(open(OUT)) if os.path.exists(OUT) else {
        "_citation": "Oracle iteration counts (oracle/amg_oracle.c via tools/oracle_golden.py); BASELINE.json configs, "
                     "SURVEY 8(d) table; relative-residual stop (reading A14)."}
    for name in names:
        p = gen.problem(name)
        t0 = time.time()
        H = oracle.setup_problem(p)
        t1 = time.time()
        r = H.solve(gen.rhs(p.n, p.params["seed"]), tol=p.params["tol"], nu=p.params["k_inner"])
        t2 = time.time()
        import numpy as np

        idx = np.unique(np.linspace(0, p.n - 1, 4096).round().astype(np.int64))
        data[name] = {"iters": r["iters"], "status": r["status"], "relres": r["relres"],
                      "x_sample_idx": idx.tolist(), "x_sample": r["x"][idx].tolist(),
                      "x_absmax": float(np.abs(r["x"]).max()), "x_norm": float(np.linalg.norm(r["x"])),
                      "true_relres": r["true_relres"], "levels": [H.level_info(l)["n"] for l in range(H.nlev)],
                      "complexities": list(H.complexities()), "oracle_setup_s": round(t1 - t0, 2),
                      "oracle_solve_s": round(t2 - t1, 2), "host": host}
        json.dump(data, open(OUT, "w"), indent=1)
        print(name, data[name], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C3"])

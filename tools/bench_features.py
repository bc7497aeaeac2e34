"""Throughput of the device row-feature pass (mpb_row_features, all five
outputs) on a BASELINE config's operator: one JSON line.

    python tools/bench_features.py [c2] [--reps 20]

Bytes per launch (algorithmic): row_ptr 4(N+1) + col_idx 4Z + values 8Z
(the row is read once; the three sums re-read it from L1) + 5 fp64 outputs
40N.  Also times the reference's numpy features (oracle restatement, one
host thread) on the same matrix for comparison."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2407_15973_b200 import _lib, problems, features as F
    from oracle import features_oracle as FO
    cs = problems.make_config(args.config)
    A = cs.A
    D = A.device()
    h = _lib.Handle.get(D.device.index)
    n, z = A.n, A.nnz
    outs = [torch.empty(n, dtype=torch.float64, device=D.device) for _ in range(5)]

    def launch():
        _lib.check(h.lib.mpb_row_features(h.ptr, n, _lib.ptr(D.row_ptr), _lib.ptr(D.col_idx), _lib.ptr(D.val64),
                                          _lib.ptr(D.val32), *[_lib.ptr(o) for o in outs]), "row_features")
    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    nbytes = 4 * (n + 1) + 12 * z + 40 * n
    t0 = time.time()
    F.dominance_stats(A), F.multiscale_histogram(A), F.m_matrix_sign_check(A)
    torch.cuda.synchronize()
    api_s = time.time() - t0
    t0 = time.time()
    tau, dfd = FO.multiscale_profile(A.row_ptr, A.col_idx, A.values)
    FO.histogram(tau, dfd, F.DECADE_EDGES), FO.dominance(A.row_ptr, A.col_idx, A.values)
    FO.sign_check(A.row_ptr, A.col_idx, A.values)
    cpu_s = time.time() - t0
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    print(json.dumps({"config": args.config, "rows": n, "nnz": z, "row_features_ms": round(ms, 4),
                      "gbs": round(nbytes / ms / 1e6, 1), "frac": round(nbytes / ms / 1e6 / peak, 4),
                      "bytes": nbytes, "api_all_three_s": round(api_s, 4),
                      "reference_numpy_all_three_s": round(cpu_s, 3)}))


if __name__ == "__main__":
    main()

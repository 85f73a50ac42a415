"""Random 6-section cascades (the reference's acceptance envelope, test_acceptance.py:39-57):
error vs the float64 oracle as 3 + 3 passes (default) and as one pass (WP_LB_MAXS=8 in a
child process); python tools/six_section_probe.py [cases] [seed]"""
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "tests"))

if len(sys.argv) > 3 and sys.argv[3] == "child":
    import torch

    import oracle
    import paper_2504_08624_b200 as wp
    from conftest import random_stable_section

    cases, seed = int(sys.argv[1]), int(sys.argv[2])
    rng = np.random.default_rng(seed)
    errs = []
    for _ in range(cases):
        f = wp.IirFilter.from_sections([random_stable_section(rng) for _ in range(6)], 44100,
                                       overall_gain=float(rng.uniform(0.25, 2.0)))
        C, N = int(rng.integers(1, 13)), int(10 ** rng.uniform(4, 5.5))
        x = rng.standard_normal((C, N)).astype(np.float32)
        y = wp.pipe(wp.Wave.from_tensor(torch.from_numpy(x).cuda(), 44100), wp.Chain([f])).tensor().cpu().numpy()
        errs.append(oracle.parity_error(y.astype(np.float64), oracle.iir_cascade(f.sos_rows(), x.astype(np.float64))))
    e = np.array(errs)
    if os.environ.get("SIX_DUMP"):
        # re-run the worst case and show where its error sits
        rng = np.random.default_rng(seed)
        for i in range(cases):
            f = wp.IirFilter.from_sections([random_stable_section(rng) for _ in range(6)], 44100,
                                           overall_gain=float(rng.uniform(0.25, 2.0)))
            C, N = int(rng.integers(1, 13)), int(10 ** rng.uniform(4, 5.5))
            x = rng.standard_normal((C, N)).astype(np.float32)
            if i != int(np.argmax(e)):
                continue
            y = wp.pipe(wp.Wave.from_tensor(torch.from_numpy(x).cuda(), 44100), wp.Chain([f])).tensor().cpu().numpy()
            ref = oracle.iir_cascade(f.sos_rows(), x.astype(np.float64))
            err = np.abs(y - ref) / np.abs(ref).max()
            c, n = np.unravel_index(np.argmax(err), err.shape)
            pos = np.arange(N) % 8192
            print(f"worst case {i}: C={C} N={N} max at ch {c} n {n} (tile pos {n % 8192}); "
                  f"mean err first 64 of tiles {err[:, pos < 64].mean():.2e}, rest {err[:, pos >= 64].mean():.2e}; "
                  f"rms(ref)/peak {np.sqrt((ref ** 2).mean()) / np.abs(ref).max():.3f}")
            np.set_printoptions(precision=4, suppress=True)
            print(f.sos_rows())
            for k, row in enumerate(f.sos_rows()):
                print(k, "pole radius", np.abs(np.roots([1, row[3], row[4]])).max().round(4),
                      "zero radii", np.abs(np.roots(row[:3])).round(3) if row[0] != 0 else "-")
    print(f"{os.environ.get('WP_LB_MAXS', 'default')}: {cases} cascades, over 1e-4: {(e > 1e-4).sum()}, "
          f"median {np.median(e):.2e}, p99 {np.percentile(e, 99):.2e}, max {e.max():.2e}")
else:
    cases = sys.argv[1] if len(sys.argv) > 1 else "1000"
    seed = sys.argv[2] if len(sys.argv) > 2 else "5"
    for maxs in (None, "8"):
        env = dict(os.environ)
        if maxs:
            env["WP_LB_MAXS"] = maxs
        subprocess.run([sys.executable, __file__, cases, seed, "child"], env=env)

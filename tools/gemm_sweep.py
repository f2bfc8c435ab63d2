"""Tall-skinny GEMM sweep over split-K and main-loop variants at the config-2 shapes."""
import json, os, subprocess, sys
shapes = [(20000, 20, 300), (20000, 20, 1200), (20000, 20, 2400), (10000, 20, 300), (10000, 20, 1200), (10000, 20, 2400)]
code = r'''
import sys, json; sys.path.insert(0, ".")
from paper_2509_21963_b200 import stages
M, N, K = map(int, sys.argv[1:4])
print(json.dumps(stages.time_gemm(M, N, K, reps=20)))
'''
for lean in ("1", "2"):
    for S in ("1", "2", "4", "8"):
        row = []
        for (M, N, K) in shapes:
            env = dict(os.environ, ITERCUR_GEMM_LEAN=lean, ITERCUR_GEMM_SPLITS=S)
            r = subprocess.run([sys.executable, "-c", code, str(M), str(N), str(K)], env=env, capture_output=True, text=True)
            try:
                us = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception:
                us = float("nan")
            bound = max(8.0 * M * K / 6452e9, 2.0 * M * 24 * K / 37.1e12) * 1e6
            row.append(f"{us:7.1f}({bound / us:4.2f})")
        print(f"lean={lean} S={S}: " + " ".join(row), flush=True)
print("shapes:", shapes)

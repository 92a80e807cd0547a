import json, sys, types
sys.path.insert(0, '.')
import bench, paper_1505_07368_b200 as pkg
ctx = pkg.Context(1)
res = bench.sec_cfg4(ctx, types.SimpleNamespace(no_cpu_baseline=False), 1)
for k, v in res.items():
    print(k, {x: v.get(x) for x in ("wall_ms", "requests_per_s", "mismatched_tiles", "good", "bad", "batches", "status")})

"""The reference harness's CSV contract for the GPU path.

`bench mandelbrot --size S --iter I --runs R --csv out.csv` (tools/bench.cpp:
113-143) appends `benchmark,param_string,workers,run_index,wall_clock_ms,
peak_rss_bytes,checksum` rows (bench.cpp:509-521). This tool runs
cafxg_run_mandelbrot the same way and appends rows with exactly those columns
(the device count goes into param_string, `workers` is 0), so reference and GPU
runs land in one file.

    python paper_1505_07368_b200/tools/bench_csv.py --size 16000 --iter 500 --runs 3 --csv out.csv
"""
import argparse
import os
import resource
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402

HEADER = "benchmark,param_string,workers,run_index,wall_clock_ms,peak_rss_bytes,checksum\n"


def main(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--size", type=int, default=16000)
    p.add_argument("--iter", type=int, default=500)
    p.add_argument("--runs", type=int, default=3)
    p.add_argument("--devices", type=int, default=0, help="device mask (0 = all)")
    p.add_argument("--csv", default="")
    a = p.parse_args(argv)
    rows = []
    with pkg.Context(a.devices) as ctx:
        ctx.run_mandelbrot(a.size, a.iter)  # warm-up (context, pools, kernels)
        for r in range(a.runs):
            chk, ms = ctx.run_mandelbrot(a.size, a.iter)
            rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1024
            rows.append(f"mandelbrot-gpu,size={a.size};iter={a.iter};devices={ctx.device_count},"
                        f"0,{r},{ms:.3f},{rss},{chk}\n")
    if a.csv:
        new = not os.path.exists(a.csv)
        with open(a.csv, "a") as f:
            if new:
                f.write(HEADER)
            f.writelines(rows)
    sys.stdout.write(HEADER + "".join(rows))


if __name__ == "__main__":
    main()

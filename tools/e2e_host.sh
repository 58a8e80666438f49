# host-side create breakdown of the benchmark batch (GPU box)
GBMW_HOST_TIMING=1 python tools/e2e_probe.py 2>&1 | grep -E "^create|run_native" | tail -6

# text-score pass counts on the config-5 data (TS_TRACE build on the box; the box copy is discarded)
SPLITQ_NVCC_EXTRA=-DTS_TRACE python -c "from paper_2605_19929_b200 import _build; _build.build(force=True)" > /dev/null 2>&1; echo build rc=$?
timeout 900 python tools/bench_c5.py 2>&1 | grep -E "TS_TRACE" | head -20

timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CD_LIB_DIR=_lib_tl timeout 120 python tools/timeline.py dc 0.9 2>&1 | tail -4
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['ms_per_step']*1e3, j['roofline']['stages'][0]['us'])"; done

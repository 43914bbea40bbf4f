python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for i in 1 2; do timeout 400 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BENCH', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"; done

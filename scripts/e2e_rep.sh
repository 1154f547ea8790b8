for i in 1 2 3; do python bench.py --no-cpu-baseline --nrhs 1 --steps 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['e2e'])"; done

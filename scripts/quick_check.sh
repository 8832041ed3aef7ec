python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --workload llama70b --no-extras --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('llama', d['us_per_step'])"
python bench.py --workload llama70b_tp8 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tp8', d['us_per_step'])"
python bench.py --workload long_context --no-extras --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('long', d['us_per_step'], d['value'])"
python bench.py --workload high_load --no-extras --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('high', d['us_per_step'], d['value'])"

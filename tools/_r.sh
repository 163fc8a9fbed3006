timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
python tools/solve_scan.py 2>&1 | grep '=='
bash tools/ab_env.sh "C5" "X=0" 2>&1 | grep -v stages_ms

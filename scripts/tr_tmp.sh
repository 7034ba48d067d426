python scripts/quick_batch.py 8192 512 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_total'], d['r0'], d['found'])"
python scripts/detect_once.py 3 2>/dev/null | tail -2
timeout 900 python -m pytest tests/test_gpu_lms.py -m gpu -x -q -k "small or batch" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_hough.py tests/test_ref_compat.py -m gpu -x -q 2>&1 | tail -2

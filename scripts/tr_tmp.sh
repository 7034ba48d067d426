timeout 600 compute-sanitizer --tool initcheck --show-backtrace no python -m pytest tests/test_gpu_lms.py -m gpu -x -q -k "deferred" 2>&1 | grep -E "Uninitialized|ERROR SUMMARY|passed|failed" | sort | uniq -c | head
timeout 1700 python -m pytest tests/test_gpu_lms.py -m gpu -q -rf 2>&1 | tail -3

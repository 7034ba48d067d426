timeout 1500 compute-sanitizer --tool memcheck --show-backtrace no python -m pytest tests/test_gpu_lms.py -m gpu -x -q -k "hybrid or deferred" 2>&1 | grep -v "Saved host" | head -30

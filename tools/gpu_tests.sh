set -x
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} 2>&1 | tail -30

cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_checked.py -q 2>&1 | tail -15

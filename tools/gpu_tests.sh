cd $GRAFT_REPO_ROOT
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} 2>&1 | tail -${TAILN:-40}

cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
TAG=f5 bash scripts/gpu.sh test smoke bench

# usage: bash scripts/lib_sweep.sh <script.py> <lib>...  -> time a script against library variants
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=$1; shift
for l in paper_1710_07193_b200/libdctf_b200.so "$@"; do echo "== $l"; DCTF_LIB_PATH=$PWD/$l timeout 300 python $S; done

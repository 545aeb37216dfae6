cd $GRAFT_REPO_ROOT
VARIANTS="compact|| union|-DP2M_COMPACT=0|" CFGS="2 5 1 4" BIGN=20000000 bash scripts/gpu_ab.sh

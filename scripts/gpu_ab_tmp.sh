VARIANTS="base|| nog1|-DP2M_NO_G1=1|" CFGS="2 2" STEPS=10 bash scripts/gpu_ab.sh 2>&1

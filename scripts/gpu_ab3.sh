VARIANTS="head|| rpw0|-DP2M_RPW=0| oldmask|-DP2M_OLD_MASK| both|-DP2M_RPW=0,-DP2M_OLD_MASK|" CFGS="2 1" STEPS=10 bash scripts/gpu_ab.sh

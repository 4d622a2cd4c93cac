cd $GRAFT_REPO_ROOT/benchmarks
MOE_B200_LIB=../exp/agather/libmoe_b200.so timeout 300 python agather_test.py
MOE_B200_LIB=../exp/agather/libmoe_b200.so timeout 300 python agather_test.py

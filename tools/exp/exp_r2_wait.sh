# mbarrier wait flavours on the d<=128 ping-pong kernel's critical path
S=2,10,0
timeout 120 python tools/exp/ab.py base $S
for v in nohint spinp spins spinps; do FMHA_B200_LIB=build/var_$v.so timeout 120 python tools/exp/ab.py $v $S; done
timeout 120 python tools/exp/ab.py base2 $S

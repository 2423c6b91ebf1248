for rep in 1 2; do
for v in noepi noepi7 epi6; do FMHA_B200_LIB=build/var_$v.so timeout 200 python tools/exp/ab.py $v 0,17,18 2>&1 | tail -3; done
timeout 200 python tools/exp/ab.py epiwg 0,17,18 2>&1 | tail -3
done
make -s prof > /dev/null 2>&1; FMHA_B200_LIB=build/libfmha_b200_prof.so python tools/prof_phases.py 16 12 512 64 2>&1 | tail -6

for rep in 1 2; do
for e in 4 6 8; do FMHA_TUNE_EMU64D=$e timeout 60 python tools/exp/ab.py e$e 1,7,8,9 2>&1 | tail -4; done
done

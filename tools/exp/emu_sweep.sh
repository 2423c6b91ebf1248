for rep in 1 2; do
for e in 0 2 4 6 8; do FMHA_TUNE_EMU=$e timeout 200 python tools/exp/ab.py emu$e 2,6,10 2>&1 | tail -3; done
done

for r in 1 2 3; do
for e in 2 4 6; do FMHA_TUNE_EMU=$e timeout 300 python tools/exp/ab.py emu$e 2,6,7; done
done

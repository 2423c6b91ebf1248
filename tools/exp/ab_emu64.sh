for r in 1 2; do
for e in 0 2 4 6; do FMHA_TUNE_EMU64=$e timeout 300 python tools/exp/ab.py emu$e 0,17,18; done
done

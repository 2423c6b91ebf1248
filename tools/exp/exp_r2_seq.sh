S=0,2,10,11,14,16
FMHA_B200_LIB=build/var_seq0.so python tools/exp/ab.py base $S
python tools/exp/ab.py seq4 $S
FMHA_TUNE_EMU=6 FMHA_TUNE_EMU64=6 python tools/exp/ab.py seq6 $S
FMHA_TUNE_EMU=8 FMHA_TUNE_EMU64=8 python tools/exp/ab.py seq8 $S
FMHA_TUNE_EMU=2 FMHA_TUNE_EMU64=4 python tools/exp/ab.py seq2 $S
FMHA_B200_LIB=build/var_seq0.so python tools/exp/ab.py base2 $S
python tools/exp/ab.py seq4b $S

for cfg in "16 512 12 64" "4 4096 16 128" "2 8192 8 256" "8 16384 32 128 bf16" "4 4096 32 64"; do
  timeout 60 build/epilogue_probe $cfg
done

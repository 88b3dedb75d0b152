mkdir -p /tmp/rep
for m in "aap 8" "et 8" "swap-push 8" "os-push 8" "os-pull 8" "aap 4" "et 4"; do set -- $m
  timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:'k_idx_aos_tiled|k_swap_idx|k_os_push_idx_aos|k_os_pull_idx_aos|k_local_idx_aos|k_local_stream|k_et_idx|k_aa_odd_idx' -c 4 -o /tmp/rep/idx_$1_$2 python tools/ncu_drive.py c4 $1 indirect aos $2 4 > gpurun_out/ncu_idx_$1_$2.log 2>&1
  ncu -i /tmp/rep/idx_$1_$2.ncu-rep --page raw --csv > gpurun_out/idx_$1_$2_raw.csv 2>&1
  ncu -i /tmp/rep/idx_$1_$2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/idx_$1_$2_src.csv 2>&1
done
du -sh gpurun_out

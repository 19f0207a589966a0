ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bwd_v2.csv python scripts/prof_attn.py > /dev/null 2>&1
AVB_LIB=$PWD/paper_2309_16669_b200/libavion_b200_expv4.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bwd_v4.csv python scripts/prof_attn.py > /dev/null 2>&1
AVB_LIB=$PWD/paper_2309_16669_b200/libavion_b200_expv4.so ncu --set full --clock-control none --import-source on -k regex:attn_bwd_d -s 2 -c 2 -o gpurun_out/bwd_v4_prof python scripts/prof_attn.py > /dev/null 2>&1
ls gpurun_out

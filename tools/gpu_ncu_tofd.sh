for lib in paper_2006_00686_b200/libxrt.so paper_2006_00686_b200/libxrt_kf.so; do
  XRT_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum -k regex:k_to_fd -c 3 python tools/time_fwd.py 4 1 2>&1 | grep -E "gpu__time_duration" | head -3
done

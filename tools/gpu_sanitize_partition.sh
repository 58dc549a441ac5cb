# compute-sanitizer over the partitioned group-by kernels (part_*_kernel).
O=gpurun_out/r02e; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --error-exitcode 9 python tools/sanitize_partition.py > $O/sanitize_partition_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -3 $O/sanitize_partition_memcheck.txt
timeout 1500 $CS --tool racecheck --racecheck-report hazard python tools/sanitize_partition.py > $O/sanitize_partition_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -3 $O/sanitize_partition_racecheck.txt
timeout 1200 $CS --tool synccheck python tools/sanitize_partition.py > $O/sanitize_partition_synccheck.txt 2>&1; echo "synccheck rc=$?"; tail -3 $O/sanitize_partition_synccheck.txt

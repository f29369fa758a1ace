for kb in 16 64 360; do for mode in 0 1 2 3; do
echo "chunk_KB $kb mode $mode: $(ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -s 1 -c 1 --csv tools/l2_reread $kb $mode 4 2>&1 | grep -E 'dram__bytes_read|gpu__time_duration|hit_rate' | awk -F'","' '{printf "%s %s %s | ", $(NF-2), $(NF-1), $NF}')"
done; done
echo "chunk 360 KB 1 cta/sm mode 0: $(ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -s 1 -c 1 --csv tools/l2_reread 360 0 1 2>&1 | grep -E 'dram__bytes_read|gpu__time_duration|hit_rate' | awk -F'","' '{printf "%s %s %s | ", $(NF-2), $(NF-1), $NF}')"

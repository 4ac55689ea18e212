for x in 0 3 4; do
SD_SCAN_EXP=$x ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sbs_scan" -s 3 -c 3 --csv --log-file gpurun_out/exp$x.csv python scripts/sweep_sparsity.py --S 50 > /dev/null 2>&1
echo "exp $x"; grep gpu__time gpurun_out/exp$x.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo
done

for v in 0 1 2; do for g in 0 32 64; do
  ./build/gather_probe g 8192 26 $v $g > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none -k regex:gather -s 1 -c 1 ./build/gather_probe g 8192 26 $v $g 2>&1 | grep -E "dram__|duration|variant" | tr '\n' ' '; echo " v=$v g=$g"
done; done

# A/B of the two-stream device many-call (lib_fk, RB_FORK_WAVES) against lib_cur: bench step value
val() { python -c "
import json; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l); print(round(d['value']/1e6,1))"; }
for c in 2 3 4 5; do
  rows=""; [ $c = 5 ] && rows="--rows 10000000"
  for v in "cur 128" "fk 0" "fk 16" "fk 128" "fk 1024"; do
    set -- $v
    RB_FORK_WAVES=$2 RB_LIB=paper_1407_7737_b200/variants/lib_$1.so timeout 600 python bench.py --config $c $rows --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/fkw_$c.txt 2>/dev/null
    echo "config $c lib $1 waves $2: $(val gpurun_out/fkw_$c.txt)"
  done
done

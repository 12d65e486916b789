val() { python -c "
import json; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l); print(round(d['value']/1e6,1))"; }
for v in "cur 128" "fk 128" "fk 16" "fk 128" "cur 128" "fk 128"; do
  set -- $v
  RB_FORK_WAVES=$2 RB_LIB=paper_1407_7737_b200/variants/lib_$1.so timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/fkw2.txt 2>/dev/null
  echo "config 2 lib $1 waves $2: $(val gpurun_out/fkw2.txt)"
done

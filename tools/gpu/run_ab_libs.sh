# interleaved A/B of two library builds (tools/lib_old.so = HEAD, the in-tree one = the working copy)
for rep in 1 2 3; do
  for lib in tools/lib_old.so paper_1002_4057_b200/libtileinv_b200.so; do
    for w in c1 c2 c3; do
      st=20; [ $w = c3 ] && st=3
      r=$(TINV_LIB=$lib timeout 300 python bench.py --workload $w --steps $st --warmup 3 --no-e2e --no-cpu --no-steps --no-load 2>/dev/null | tail -1)
      echo "$lib $w $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d.get("kernel_ms",0),3))')"
    done
  done
done

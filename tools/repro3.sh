python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -c "import paper_1610_05994_b200 as wt; print(wt.launch_plan(8000000, 1<<24, 4))" > gpurun_out/plan5.txt
for args in "5 2000000" "5 4000000" "5 8000000" "4 16000000" "4 40000000"; do
  WT_DEBUG_SYNC=1 timeout 300 python tools/repro2.py $args >> gpurun_out/repro3.log 2>&1
done

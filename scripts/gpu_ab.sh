mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ARGS="--steps 50 --no-cpu-baseline --no-e2e --no-clocks"
(cd _old && python -m paper_1909_03355_b200.build > /dev/null 2>&1)
(cd _old && python bench.py $ARGS > ../gpurun_out/ab_old.json 2>../gpurun_out/ab_old.err) && echo oldok
python bench.py $ARGS > gpurun_out/ab_new.json 2>gpurun_out/ab_new.err && echo newok
(cd _old && timeout 600 ncu --set full --import-source on --kernel-name regex:node_kernel --launch-skip 5 -c 1 -o ../gpurun_out/node_old -f python bench.py $ARGS > ../gpurun_out/ncu_old.log 2>&1); echo ncuold=$?
timeout 600 ncu --set full --import-source on --kernel-name regex:node_kernel --launch-skip 5 -c 1 -o gpurun_out/node_new -f python bench.py $ARGS > gpurun_out/ncu_new.log 2>&1; echo ncunew=$?
timeout 900 ncu --set full --import-source on --kernel-name regex:element_chunk --launch-skip 5 -c 1 -o gpurun_out/elem_new -f python bench.py $ARGS > gpurun_out/ncu_elem.log 2>&1; echo ncuelem=$?

# r02z36: C3 step with prep_b beside entangle and recover beside check (second stream) vs strictly in order, alternating
O=gpurun_out/r02z36; mkdir -p $O
for k in 1 2; do
for ov in 0 1; do
timeout 600 python bench.py --configs 0 --workload c3 --overlap $ov > $O/b_c3_ov${ov}_$k.json 2> $O/b_c3_ov${ov}_$k.err; echo ov$ov rc=$?
python -c "import json; d=json.load(open('$O/b_c3_ov${ov}_$k.json')); print('overlap $ov', d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['correctness']['oracle_rows_equal'], d['launch'])"
done; done

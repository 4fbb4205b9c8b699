for rep in 1 2; do
timeout 300 python -c "
import json, bench, torch
import paper_2509_18172_b200 as sb
print(json.dumps(bench.layer_chain(sb, torch.device('cuda'))))
" 2>&1 | tail -1
done

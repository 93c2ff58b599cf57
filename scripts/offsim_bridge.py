"""Feed the measured B200 costs into the reference simulator (runs where the reference
is importable: this container, PYTHONPATH=/root/reference/pkg/src).

* profiles/b200_cost_table.csv (measured by scripts/export_cost_table.py on the GPU)
  replaces indexer_logits / indexer_topk / sparse_mla / merge_attn of the reference's
  calibrated profile (offsim.profiles.calibrated_profile; the ops outside this repo's
  path keep their calibrated values) -> profiles/b200_cost_table_full.csv;
* profiles/b200_cost_table.transfer.json (the measured K4 gather rate) becomes the
  scenario's [transfer] section -> profiles/b200_transfer.toml;
* offsim.pipeline.simulate_decode is run on the default scenario with the shipped
  profile and with the B200 one, and the predicted iteration time / throughput printed.
"""
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("OFFSIM_SRC", "/root/reference/pkg/src"))

from offsim import costmodel, pipeline, profiles, scenario, trace  # noqa: E402

from paper_2512_10576_b200 import costbridge  # noqa: E402

PROF = os.path.join(ROOT, "profiles")
measured = costbridge.read_cost_table(os.path.join(PROF, "b200_cost_table.csv"))
with open(os.path.join(PROF, "b200_cost_table.transfer.json")) as f:
    tcfg = json.load(f)
s = scenario.default_scenario()
base = profiles.calibrated_profile(mtp=s.model.mtp_width, context=32768, model=s.model).table
with tempfile.TemporaryDirectory() as d:
    costmodel.save_cost_table(base, os.path.join(d, "base.csv"))
    base_entries = costbridge.read_cost_table(os.path.join(d, "base.csv"))
full = costbridge.merge_cost_tables(measured, base_entries)
full_path = os.path.join(PROF, "b200_cost_table_full.csv")
costbridge.write_cost_table(full, full_path)
with open(os.path.join(PROF, "b200_transfer.toml"), "w") as f:
    f.write("# measured on B200 (scripts/export_cost_table.py): K4 zero-copy gather of 656-B rows\n")
    f.write("[transfer]\n")
    for k, v in tcfg.items():
        f.write(f"{k} = {json.dumps(v)}\n")
table = costmodel.load_cost_table(full_path)          # the reference's own loader
transfer = costmodel.TransferModel.from_dict(tcfg)    # and its own [transfer] parser
tr = trace.generate_trace(trace.TraceGenParams(num_layers=s.model.num_layers, context_len=s.deploy.context_len,
                                               topk=s.effective_topk(), num_steps=4,
                                               target_similarity=0.9,
                                               mean_accept=s.model.accept_ratio, seed=0))
for name, tab, tm in (("shipped calibrated profile", base, costmodel.TransferModel()),
                      ("B200 measured profile", table, transfer)):
    r = pipeline.simulate_decode(s, tr, tab, tm)
    print(f"{name:28s} mean_iter_us={r.mean_iter_us:9.1f} otps={r.otps:8.2f} throughput={r.throughput:10.1f}")
print("->", full_path)

"""Generate the committed Himeno program model with the *reference* front-end.

Runs in the dev container only (needs /root/reference): parses the Himeno
C-subset text (apps/himeno.py) with acctuner.code_model.analyze_project,
classifies it with acctuner.classify.StaticRuleProbe, and writes
paper_2002_12115_b200/apps/model/himeno.json = the reference's structural JSON
(dump_structural) + index_var_keys + the classifier verdicts.  The structure
is checked to be identical across XS/M/L/XL (only spans/trip counts differ).

    PYTHONPATH=/root/reference/pkg/src python scripts/gen_program_model.py
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from acctuner.classify import StaticRuleProbe, classify_project, eligible_ids  # noqa: E402
from acctuner.code_model import analyze_project, dump_structural  # noqa: E402

from paper_2002_12115_b200.apps import ft, himeno  # noqa: E402


def analyze(size_name, nn=3):
    sz = himeno.size(size_name)
    fid = himeno.source_file_id(sz)
    proj = analyze_project([(fid, himeno.source_text(sz, nn))])
    verdicts = classify_project(proj, StaticRuleProbe())
    doc = dump_structural(proj)
    doc["index_var_keys"] = sorted(proj.refs.index_var_keys)
    doc["verdicts"] = [v.to_json() for v in verdicts]
    doc["eligible"] = eligible_ids(verdicts)
    return doc


def shape_only(doc):
    out = json.loads(json.dumps(doc))
    for f in out["files"]:
        f["file_id"] = "_"
        for l in f["loops"]:
            l["span"] = None
            l["trip_count"] = None
        for v in f["vars"]:
            v.pop("extent", None)
    return out


def analyze_ft(cls_name):
    c = ft.ft_class(cls_name)
    proj = analyze_project([(ft.source_file_id(c), ft.source_text(c))])
    verdicts = classify_project(proj, StaticRuleProbe())
    doc = dump_structural(proj)
    doc["index_var_keys"] = sorted(proj.refs.index_var_keys)
    doc["verdicts"] = [v.to_json() for v in verdicts]
    doc["eligible"] = eligible_ids(verdicts)
    doc["generated_by"] = (f"scripts/gen_program_model.py: reference acctuner analyze_project + "
                           f"StaticRuleProbe on ft.source_text('{c.name}')")
    return doc


def main_ft():
    for name in ("S", "W", "A"):
        doc = analyze_ft(name)
        out = ROOT / "paper_2002_12115_b200" / "apps" / "model" / f"ft_{name.lower()}.json"
        out.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
        print(f"wrote {out}: {sum(len(f['loops']) for f in doc['files'])} loops, "
              f"gene length {len(doc['eligible'])}")


def main():
    main_ft()
    base = analyze("XS")
    for name in ("M", "L", "XL"):
        if shape_only(analyze(name)) != shape_only(base):
            raise SystemExit(f"structure of {name} differs from XS")
    base["generated_by"] = ("scripts/gen_program_model.py: reference acctuner "
                            "analyze_project + StaticRuleProbe on himeno.source_text('XS', 3)")
    out = ROOT / "paper_2002_12115_b200" / "apps" / "model" / "himeno.json"
    out.write_text(json.dumps(base, indent=1, sort_keys=True) + "\n")
    print(f"wrote {out}: {sum(len(f['loops']) for f in base['files'])} loops, "
          f"gene length {len(base['eligible'])}")


if __name__ == "__main__":
    main()

import paper_2112_14064_b200 as rq
rq.baseline_config("cfg4_riga", device=True, resident=True)

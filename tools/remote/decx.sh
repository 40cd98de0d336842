python tools/decode_exp.py base
cp paper_2603_21365_b200/_lib/libtide_b200.so /tmp/base.so
for e in 1 2 3 4; do cp tools/_libs/dec$e.so paper_2603_21365_b200/_lib/libtide_b200.so; python tools/decode_exp.py exp$e; done
cp /tmp/base.so paper_2603_21365_b200/_lib/libtide_b200.so

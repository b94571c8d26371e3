cd $GRAFT_REPO_ROOT
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
cp paper_2405_00698_b200/_lib_debug/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so

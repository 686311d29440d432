bash tools/gpujob_ab.sh cur redb C2 1024
bash tools/gpujob_ab.sh cur redb C4 64

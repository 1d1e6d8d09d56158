# per-layer fwd / bwd times (one stage, serialised backward) of VGG-16 and the LSTM LM
TAG=${TAG:-r2lp}; mkdir -p gpurun_out/$TAG
for w in vgg16 lstm_lm; do timeout 300 python tools/layer_prof.py $w > gpurun_out/$TAG/$w.jsonl 2>&1; done

import pynvml, torch
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for fid in (138, 139, 140, 141):
    try:
        v = pynvml.nvmlDeviceGetFieldValues(h, [fid])[0]
        print(fid, 'ret', v.nvmlReturn, 'type', v.valueType, 'ull', v.value.ullVal, 'scope', v.scopeId)
    except Exception as e:
        print(fid, 'exc', e)
# per-link with scopeId
try:
    fv = pynvml.c_nvmlFieldValue_t * 2
    vals = fv(); vals[0].fieldId = 138; vals[0].scopeId = 0; vals[1].fieldId = 138; vals[1].scopeId = 1
    r = pynvml.nvmlDeviceGetFieldValues(h, [138])
    print('ok list')
except Exception as e: print('exc2', e)
try:
    print('util counter', pynvml.nvmlDeviceGetNvLinkUtilizationCounter(h, 0, 0))
except Exception as e: print('util exc', e)

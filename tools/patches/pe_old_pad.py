# previous (staged) patch-embed kernel with its positional slice rows padded by 16 bytes
p = 'paper_2511_22009_b200/csrc/dit_runtime.cu'
s = open(p).read()
s = s.replace("static constexpr int POS = 16 * HID * 4;", "static constexpr int POS = 16 * (HID + 4) * 4;")
s = s.replace("reinterpret_cast<float4*>(sPos)[idx] = make_float4(", "reinterpret_cast<float4*>(sPos + r * (HID + 4))[c4] = make_float4(")
s = s.replace("const float* pos0 = sPos + g * HID + 8 * c;\n  const float* pos1 = pos0 + 8 * HID;",
              "const float* pos0 = sPos + g * (HID + 4) + 8 * c;\n  const float* pos1 = pos0 + 8 * (HID + 4);")
assert s.count("(HID + 4)") == 4, s.count("(HID + 4)")
open(p, 'w').write(s)

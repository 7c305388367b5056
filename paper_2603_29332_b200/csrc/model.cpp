// Model/clip ingest and the model compiler (see model.hpp).
#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <set>
#include <sstream>

#include <json.hpp>

namespace msk_b200 {

using Json = nlohmann::json;

namespace {

void only_keys(const Json& o, std::initializer_list<const char*> allowed, const std::string& where) {
    if (!o.is_object()) throw ConfigError(where + ": expected an object");
    for (auto it = o.begin(); it != o.end(); ++it) {
        bool ok = false;
        for (const char* k : allowed) ok = ok || it.key() == k;
        if (!ok) throw ConfigError(where + ": unknown key '" + it.key() + "'");
    }
}

double num(const Json& o, const char* key, const std::string& where) {
    if (!o.contains(key)) throw ConfigError(where + ": missing key '" + key + "'");
    if (!o[key].is_number()) throw ConfigError(where + ": key '" + key + "' must be a number");
    return o[key].get<double>();
}

double num_or(const Json& o, const char* key, double dflt) {
    return o.contains(key) ? o[key].get<double>() : dflt;
}

std::string str(const Json& o, const char* key, const std::string& where) {
    if (!o.contains(key)) throw ConfigError(where + ": missing key '" + key + "'");
    if (!o[key].is_string()) throw ConfigError(where + ": key '" + key + "' must be a string");
    return o[key].get<std::string>();
}

void xz(const Json& j, const std::string& where, double& x, double& z) {
    if (!j.is_array() || j.size() != 2) throw ConfigError(where + ": expected [x, z]");
    x = j[0].get<double>();
    z = j[1].get<double>();
}

}  // namespace

std::vector<std::string> ModelSpec::validate() const {
    // Same invariants as ModelSpec::validate (model.cpp:18-86).
    std::vector<std::string> e;
    const int nl = static_cast<int>(links.size()), nj = static_cast<int>(joints.size());
    if (links.empty()) e.push_back("model has no links");
    for (const auto& l : links) {
        if (!(l.mass > 0.0)) e.push_back("link '" + l.name + "': mass must be > 0");
        if (!(l.inertia > 0.0)) e.push_back("link '" + l.name + "': inertia must be > 0");
        if (!(l.length > 0.0)) e.push_back("link '" + l.name + "': length must be > 0");
    }
    const int want = floating ? nl - 1 : nl;
    if (nj != want)
        e.push_back("expected " + std::to_string(want) + " joints for " + std::to_string(nl) + " links, got " +
                    std::to_string(nj));
    const int fc = floating ? 1 : 0;
    for (int j = 0; j < nj; ++j) {
        const auto& t = joints[j];
        if (t.child != fc + j) e.push_back("joint '" + t.name + "': joints must be listed in child-link order");
        if (t.parent >= t.child) e.push_back("joint '" + t.name + "': parent must precede child");
        if (t.parent < -1 || t.parent >= nl) e.push_back("joint '" + t.name + "': parent link out of range");
        if (t.parent == -1 && (floating || j != 0))
            e.push_back("joint '" + t.name + "': world parent only valid for the first fixed-base joint");
        if (!(t.lo < t.hi)) e.push_back("joint '" + t.name + "': limit_lo must be < limit_hi");
        if (t.damping < 0.0) e.push_back("joint '" + t.name + "': damping must be >= 0");
    }
    for (const auto& m : muscles) {
        if (!(m.f_max > 0.0)) e.push_back("muscle '" + m.name + "': f_max must be > 0");
        if (!(m.l_opt > 0.0)) e.push_back("muscle '" + m.name + "': l_opt must be > 0");
        if (!(m.v_max > 0.0)) e.push_back("muscle '" + m.name + "': v_max must be > 0");
        if (!(m.tau_act > 0.0 && m.tau_act <= m.tau_deact))
            e.push_back("muscle '" + m.name + "': need 0 < tau_act <= tau_deact");
        if (m.slack < 0.0) e.push_back("muscle '" + m.name + "': tendon_slack must be >= 0");
        if (m.vias.size() < 2) e.push_back("muscle '" + m.name + "': needs at least 2 via points");
        std::set<int> spanned;
        for (const auto& v : m.vias) {
            if (v.link < -1 || v.link >= nl)
                e.push_back("muscle '" + m.name + "': via point references missing link " + std::to_string(v.link));
            spanned.insert(v.link);
        }
        if (spanned.size() < 2) e.push_back("muscle '" + m.name + "': via points must span at least 2 distinct links");
        if (floating && spanned.count(-1))
            e.push_back("muscle '" + m.name + "': floating-root models cannot anchor muscles to the world");
    }
    for (const auto& s : spheres) {
        if (s.link < 0 || s.link >= nl) e.push_back("contact sphere references missing link");
        if (!(s.radius > 0.0)) e.push_back("contact sphere radius must be > 0");
    }
    for (int k : key_bodies)
        if (k < 0 || k >= nl) e.push_back("key body index out of range");
    if (c_k < 0 || c_c < 0 || c_mu < 0 || c_vs < 0) e.push_back("contact parameters must be >= 0");
    return e;
}

std::vector<std::string> ModelSpec::device_envelope() const {
    // What msk_gpu_create enforces.  The reference steps any model load_model
    // parses (load_model, model.cpp:198-204, and Env::Env, env.cpp:74-87, never
    // call validate), so only the structure the device tables are built from is
    // required here: the joint/child ordering of the tree (FK, the level schedule
    // and the articulated-body passes assume parents precede children), link
    // indices in range, and no world anchors on a floating root (the device keeps
    // geometry root-relative).  Physical-range checks (masses, limits, damping,
    // tau_act <= tau_deact, ...) stay in validate() / msk_gpu_validate.
    std::vector<std::string> e;
    const int nl = static_cast<int>(links.size()), nj = static_cast<int>(joints.size());
    if (links.empty()) e.push_back("model has no links");
    const int want = floating ? nl - 1 : nl;
    if (nj != want)
        e.push_back("expected " + std::to_string(want) + " joints for " + std::to_string(nl) + " links, got " +
                    std::to_string(nj));
    const int fc = floating ? 1 : 0;
    for (int j = 0; j < nj; ++j) {
        const auto& t = joints[j];
        if (t.child != fc + j) e.push_back("joint '" + t.name + "': joints must be listed in child-link order");
        if (t.parent >= t.child) e.push_back("joint '" + t.name + "': parent must precede child");
        if (t.parent < -1 || t.parent >= nl) e.push_back("joint '" + t.name + "': parent link out of range");
        if (t.parent == -1 && floating)
            e.push_back("joint '" + t.name + "': floating-root models have no world-parented joints on the device");
    }
    for (const auto& m : muscles)
        for (const auto& v : m.vias) {
            if (v.link < -1 || v.link >= nl)
                e.push_back("muscle '" + m.name + "': via point references missing link " + std::to_string(v.link));
            if (floating && v.link == -1)
                e.push_back("muscle '" + m.name + "': floating-root models cannot anchor muscles to the world");
        }
    for (const auto& s : spheres)
        if (s.link < 0 || s.link >= nl) e.push_back("contact sphere references missing link");
    for (int k : key_bodies)
        if (k < 0 || k >= nl) e.push_back("key body index out of range");
    return e;
}

ModelSpec load_model(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError("model: cannot open '" + path + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    Json root;
    try {
        root = Json::parse(ss.str());
    } catch (const Json::parse_error& ex) {
        throw ConfigError(path + ": " + ex.what());
    }
    // Key set of parse_model_json (model.cpp:96-99); "contact_spheres" is
    // accepted but ignored there, and here.
    only_keys(root, {"name", "root", "gravity", "joint_limit_stiffness", "links", "joints", "muscles", "contacts",
                     "contact_spheres", "key_bodies"},
              path);
    ModelSpec s;
    s.name = str(root, "name", path);
    const std::string rt = str(root, "root", path);
    if (rt == "fixed")
        s.floating = false;
    else if (rt == "floating")
        s.floating = true;
    else
        throw ConfigError(path + ": root must be 'fixed' or 'floating'");
    s.gravity = num_or(root, "gravity", -9.81);
    s.k_lim = num_or(root, "joint_limit_stiffness", 200.0);
    if (!root.contains("links")) throw ConfigError(path + ": missing key 'links'");
    for (const auto& jl : root["links"]) {
        only_keys(jl, {"name", "length", "mass", "inertia", "com"}, path + ".links");
        LinkSpec l;
        l.name = str(jl, "name", path + ".links");
        l.length = num(jl, "length", l.name);
        l.mass = num(jl, "mass", l.name);
        l.inertia = num(jl, "inertia", l.name);
        l.com = num(jl, "com", l.name);
        s.links.push_back(l);
    }
    if (root.contains("joints"))
        for (const auto& jj : root["joints"]) {
            only_keys(jj, {"name", "child", "parent", "anchor", "mount_angle", "limits", "damping"}, path + ".joints");
            JointSpec t;
            t.name = str(jj, "name", path + ".joints");
            t.child = static_cast<int>(num(jj, "child", t.name));
            t.parent = static_cast<int>(num(jj, "parent", t.name));
            if (!jj.contains("anchor")) throw ConfigError(t.name + ".anchor: expected [x, z]");
            xz(jj["anchor"], t.name + ".anchor", t.ax, t.az);
            t.mount = num_or(jj, "mount_angle", 0.0);
            if (jj.contains("limits")) {
                t.lo = jj["limits"][0].get<double>();
                t.hi = jj["limits"][1].get<double>();
            }
            t.damping = num_or(jj, "damping", 0.0);
            s.joints.push_back(t);
        }
    if (root.contains("muscles"))
        for (const auto& jm : root["muscles"]) {
            only_keys(jm, {"name", "f_max", "l_opt", "v_max", "tau_act", "tau_deact", "tendon_slack", "via_points"},
                      path + ".muscles");
            MuscleSpec m;
            m.name = str(jm, "name", path + ".muscles");
            m.f_max = num(jm, "f_max", m.name);
            m.l_opt = num(jm, "l_opt", m.name);
            m.v_max = num_or(jm, "v_max", 10.0);
            m.tau_act = num_or(jm, "tau_act", 0.010);
            m.tau_deact = num_or(jm, "tau_deact", 0.040);
            m.slack = num(jm, "tendon_slack", m.name);
            if (!jm.contains("via_points")) throw ConfigError(m.name + ": missing via_points");
            for (const auto& vp : jm["via_points"]) {
                if (!vp.is_array() || vp.size() != 2) throw ConfigError(m.name + ": via point must be [link, [x, z]]");
                Via v;
                v.link = vp[0].get<int>();
                xz(vp[1], m.name + ".via_point", v.x, v.z);
                m.vias.push_back(v);
            }
            s.muscles.push_back(m);
        }
    if (root.contains("contacts")) {
        const auto& jc = root["contacts"];
        only_keys(jc, {"stiffness", "damping", "friction", "smoothing_vel", "spheres"}, path + ".contacts");
        s.c_k = num_or(jc, "stiffness", s.c_k);
        s.c_c = num_or(jc, "damping", s.c_c);
        s.c_mu = num_or(jc, "friction", s.c_mu);
        s.c_vs = num_or(jc, "smoothing_vel", s.c_vs);
        if (jc.contains("spheres"))
            for (const auto& js : jc["spheres"]) {
                only_keys(js, {"link", "offset", "radius"}, path + ".contacts.spheres");
                SphereSpec sp;
                sp.link = static_cast<int>(num(js, "link", "sphere"));
                if (!js.contains("offset")) throw ConfigError("sphere.offset: expected [x, z]");
                xz(js["offset"], "sphere.offset", sp.x, sp.z);
                sp.radius = num(js, "radius", "sphere");
                s.spheres.push_back(sp);
            }
    }
    if (root.contains("key_bodies"))
        for (const auto& kb : root["key_bodies"]) s.key_bodies.push_back(kb.get<int>());
    return s;
}

Clip load_clip(const std::string& path, const ModelSpec& spec) {
    std::ifstream in(path);
    if (!in) throw ConfigError("csv: cannot open '" + path + "'");
    std::string line;
    if (!std::getline(in, line)) throw ConfigError("csv: empty file '" + path + "'");
    if (!line.empty() && line.back() == '\r') line.pop_back();
    auto split = [](const std::string& l) {
        std::vector<std::string> out;
        std::string f;
        std::istringstream is(l);
        while (std::getline(is, f, ',')) out.push_back(f);
        if (!l.empty() && l.back() == ',') out.push_back("");
        return out;
    };
    const std::vector<std::string> cols = split(line);
    std::vector<double> vals;
    int rows = 0;
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        const auto f = split(line);
        if (f.size() != cols.size())
            throw ConfigError("csv: row " + std::to_string(rows + 1) + " of '" + path + "' has " +
                              std::to_string(f.size()) + " fields, expected " + std::to_string(cols.size()));
        for (const auto& s : f) {
            try {
                vals.push_back(std::stod(s));
            } catch (const std::exception&) {
                throw ConfigError("csv: non-numeric field '" + s + "' in '" + path + "'");
            }
        }
        ++rows;
    }
    if (rows < 1) throw ConfigError("reference '" + path + "' has no frames");
    const size_t nc = cols.size();
    auto at = [&](int r, size_t c) { return vals[static_cast<size_t>(r) * nc + c]; };
    size_t c = 0;
    auto expect = [&](const std::string& name) {
        if (c >= nc || cols[c] != name)
            throw ConfigError("reference '" + path + "': expected column '" + name + "' at position " +
                              std::to_string(c));
        return c++;
    };
    Clip clip;
    clip.frames = rows;
    clip.nq = spec.nq();
    clip.nk = static_cast<int>(spec.key_bodies.size());
    const size_t tc = expect("time");
    if (rows >= 2) {
        const double dt = at(1, tc) - at(0, tc);
        if (dt > 0) clip.rate = 1.0 / dt;
    }
    const int nq = clip.nq, nk = clip.nk;
    clip.q.resize(static_cast<size_t>(rows) * nq);
    clip.dq.resize(static_cast<size_t>(rows) * nq);
    clip.key_pos.resize(static_cast<size_t>(rows) * 2 * nk);
    clip.key_angle.resize(static_cast<size_t>(rows) * nk);
    for (int j = 0; j < nq; ++j) {
        const size_t cc = expect("q_" + std::to_string(j));
        for (int r = 0; r < rows; ++r) clip.q[static_cast<size_t>(r) * nq + j] = at(r, cc);
    }
    for (int j = 0; j < nq; ++j) {
        const size_t cc = expect("dq_" + std::to_string(j));
        for (int r = 0; r < rows; ++r) clip.dq[static_cast<size_t>(r) * nq + j] = at(r, cc);
    }
    for (int k = 0; k < nk; ++k) {
        const size_t cx = expect("key" + std::to_string(k) + "_x");
        const size_t cz = expect("key" + std::to_string(k) + "_z");
        for (int r = 0; r < rows; ++r) {
            clip.key_pos[static_cast<size_t>(r) * 2 * nk + 2 * k] = at(r, cx);
            clip.key_pos[static_cast<size_t>(r) * 2 * nk + 2 * k + 1] = at(r, cz);
        }
    }
    for (int k = 0; k < nk; ++k) {
        const size_t ca = expect("key" + std::to_string(k) + "_angle");
        for (int r = 0; r < rows; ++r) clip.key_angle[static_cast<size_t>(r) * nk + k] = at(r, ca);
    }
    int n_emg = 0;
    while (c + n_emg < nc && cols[c + n_emg] == "emg_" + std::to_string(n_emg)) ++n_emg;
    clip.n_emg = n_emg;
    clip.emg.resize(static_cast<size_t>(rows) * n_emg);
    for (int e = 0; e < n_emg; ++e)
        for (int r = 0; r < rows; ++r) clip.emg[static_cast<size_t>(r) * n_emg + e] = at(r, c + e);
    c += n_emg;
    int n_grf = 0;
    while (c + 2 * n_grf + 1 < nc && cols[c + 2 * n_grf] == "grf" + std::to_string(n_grf) + "_x") ++n_grf;
    c += 2 * n_grf;  // GRF columns are logged, never read by the step path
    if (c != nc) throw ConfigError("reference '" + path + "': unexpected column '" + cols[c] + "'");
    // ReferenceTrajectory::validate (reference.cpp:11-33)
    if (rows < 2) throw ConfigError("reference '" + path + "': reference needs at least 2 frames");
    if (std::abs(clip.rate * 0.02 - 1.0) > 1e-9)
        throw ConfigError("reference '" + path + "': reference rate must be 50 Hz (control rate)");
    for (const auto* v : {&clip.q, &clip.dq, &clip.key_pos, &clip.key_angle})
        for (double x : *v)
            if (!std::isfinite(x)) throw ConfigError("reference '" + path + "': reference contains non-finite values");
    return clip;
}

CompiledModel compile_model(const ModelSpec& s) {
    CompiledModel c;
    c.floating = s.floating ? 1 : 0;
    c.nl = static_cast<int>(s.links.size());
    c.nj = static_cast<int>(s.joints.size());
    c.nrd = s.nrd();
    c.nq = s.nq();
    c.nm = static_cast<int>(s.muscles.size());
    c.nk = static_cast<int>(s.key_bodies.size());
    c.ns = static_cast<int>(s.spheres.size());
    c.gravity = static_cast<float>(s.gravity);
    c.k_lim = static_cast<float>(s.k_lim);
    c.k_lim_d = s.k_lim;
    c.c_k = static_cast<float>(s.c_k);
    c.c_c = static_cast<float>(s.c_c);
    c.c_mu = static_cast<float>(s.c_mu);
    c.inv_c_vs = static_cast<float>(1.0 / s.c_vs);
    const int fc = c.floating;
    // links
    c.link_parent.assign(c.nl, -1);
    c.link_dof.assign(c.nl, -1);
    c.link_ax.assign(c.nl, 0.f);
    c.link_az.assign(c.nl, 0.f);
    c.link_mount.assign(c.nl, 0.0);
    for (int j = 0; j < c.nj; ++j) {
        const int l = fc + j;
        c.link_parent[l] = s.joints[j].parent;
        c.link_dof[l] = c.nrd + j;
        c.link_ax[l] = static_cast<float>(s.joints[j].ax);
        c.link_az[l] = static_cast<float>(s.joints[j].az);
        c.link_mount[l] = s.joints[j].mount;
        c.joint_damping.push_back(static_cast<float>(s.joints[j].damping));
        c.joint_lo.push_back(s.joints[j].lo);
        c.joint_hi.push_back(s.joints[j].hi);
    }
    for (const auto& l : s.links) {
        c.link_com.push_back(static_cast<float>(l.com));
        c.link_mass.push_back(static_cast<float>(l.mass));
        c.link_inertia.push_back(static_cast<float>(l.inertia));
    }
    // depth levels (parents precede children, so one pass suffices)
    std::vector<int> depth(c.nl, 0);
    for (int l = 0; l < c.nl; ++l) depth[l] = c.link_parent[l] >= 0 ? depth[c.link_parent[l]] + 1 : 0;
    const int maxd = c.nl ? *std::max_element(depth.begin(), depth.end()) : 0;
    c.n_levels = maxd + 1;
    c.level_start.assign(c.n_levels + 1, 0);
    for (int d = 0; d <= maxd; ++d) {
        c.level_start[d] = static_cast<int>(c.level_links.size());
        for (int l = 0; l < c.nl; ++l)
            if (depth[l] == d) c.level_links.push_back(l);
    }
    c.level_start[c.n_levels] = static_cast<int>(c.level_links.size());
    c.child_start.assign(c.nl + 1, 0);
    for (int l = 0; l < c.nl; ++l) {
        c.child_start[l] = static_cast<int>(c.child_list.size());
        for (int k = 0; k < c.nl; ++k)
            if (c.link_parent[k] == l) c.child_list.push_back(k);
    }
    c.child_start[c.nl] = static_cast<int>(c.child_list.size());
    c.sphere_start.assign(c.nl + 1, 0);
    for (int l = 0; l < c.nl; ++l) {
        c.sphere_start[l] = static_cast<int>(c.sphere_x.size());
        for (const auto& sp : s.spheres)
            if (sp.link == l) {
                c.sphere_x.push_back(static_cast<float>(sp.x));
                c.sphere_z.push_back(static_cast<float>(sp.z));
                c.sphere_r.push_back(static_cast<float>(sp.radius));
                c.sphere_link.push_back(l);
            }
    }
    c.sphere_start[c.nl] = static_cast<int>(c.sphere_x.size());
    // muscles
    const double dt = 0.002;
    auto path = [&](int link) {
        std::vector<int> p;
        int cur = link;
        while (cur >= fc) {
            p.push_back(cur - fc);
            cur = s.joints[cur - fc].parent;
        }
        return p;
    };
    struct Pair {
        int joint, via, muscle;
        float sign;
        int seg;  // adjacent segment owning this pair, or -1 (general pair)
    };
    std::vector<Pair> pairs;
    c.m_via_start.push_back(0);
    c.m_pair_start.push_back(0);
    c.m_seg_start.push_back(0);
    auto parent_of = [&](int link) { return link >= fc ? s.joints[link - fc].parent : -2; };
    for (int mi = 0; mi < c.nm; ++mi) {
        const auto& m = s.muscles[mi];
        c.m_fmax.push_back(static_cast<float>(m.f_max));
        c.m_lopt.push_back(m.l_opt);
        c.m_inv_lopt.push_back(1.0 / m.l_opt);
        c.m_slack.push_back(m.slack);
        c.m_kv.push_back(1.0 / (dt * m.l_opt * m.v_max));
        // exp(-dt/tau) is evaluated as exp2: the constants carry log2(e)
        c.m_ndt_act.push_back(static_cast<float>(-dt / m.tau_act * 1.4426950408889634));
        c.m_ndt_deact.push_back(static_cast<float>(-dt / m.tau_deact * 1.4426950408889634));
        c.m_pw.push_back(static_cast<float>(m.l_opt * m.v_max / 10.0));
        const int v0 = static_cast<int>(c.via_link.size());
        for (const auto& v : m.vias) {
            c.via_link.push_back(v.link);
            c.via_x.push_back(static_cast<float>(v.x));
            c.via_z.push_back(static_cast<float>(v.z));
        }
        c.max_via = std::max(c.max_via, static_cast<int>(m.vias.size()));
        c.m_via_start.push_back(static_cast<int>(c.via_link.size()));
        // J_m^T F through the joints between a segment's two links: joints on
        // only one side of the tree path see the segment force; common
        // ancestors (and the floating root) see a zero net wrench.
        for (int k = 1; k < static_cast<int>(m.vias.size()); ++k) {
            const Via& va = m.vias[k - 1];
            const Via& vb = m.vias[k];
            const int la = va.link, lb = vb.link;
            const int seg = static_cast<int>(c.seg_info.size());
            if (la == lb) {  // rigid: constant length, no net wrench
                c.seg_info.push_back(0);
                c.seg_slot.push_back(-1);
                c.seg_ax.push_back(static_cast<float>(std::hypot(vb.x - va.x, vb.z - va.z)));
                c.seg_az.push_back(0.f);
                c.seg_cx.push_back(0.f);
                c.seg_cz.push_back(0.f);
                continue;
            }
            const bool b_child = lb >= 0 && parent_of(lb) == la;
            const bool a_child = la >= 0 && parent_of(la) == lb;
            if (b_child || a_child) {  // adjacent: evaluate in the parent's frame
                const int child = b_child ? lb : la;
                const Via& vp = b_child ? va : vb;
                const Via& vc = b_child ? vb : va;
                const auto& jt = s.joints[child - fc];
                c.seg_info.push_back(1 | ((c.nrd + child - fc) << 8));
                c.seg_slot.push_back(-1);  // filled once slots are assigned
                c.seg_ax.push_back(static_cast<float>(jt.ax - vp.x));
                c.seg_az.push_back(static_cast<float>(jt.az - vp.z));
                c.seg_cx.push_back(static_cast<float>(vc.x));
                c.seg_cz.push_back(static_cast<float>(vc.z));
                pairs.push_back({child - fc, v0 + k, mi, b_child ? -1.0f : +1.0f, seg});
                continue;
            }
            c.seg_info.push_back(2);
            c.seg_slot.push_back(v0 + k);
            c.seg_ax.push_back(0.f);
            c.seg_az.push_back(0.f);
            c.seg_cx.push_back(0.f);
            c.seg_cz.push_back(0.f);
            const auto pa = path(la), pb = path(lb);
            std::set<int> sa(pa.begin(), pa.end()), sb(pb.begin(), pb.end());
            for (int j : sb)
                if (!sa.count(j)) pairs.push_back({j, v0 + k, mi, -1.0f, -1});
            for (int j : sa)
                if (!sb.count(j)) pairs.push_back({j, v0 + k, mi, +1.0f, -1});
        }
        c.m_seg_start.push_back(static_cast<int>(c.seg_info.size()));
        int n_general = 0;
        for (const auto& p : pairs)
            if (p.seg < 0) ++n_general;
        c.m_pair_start.push_back(n_general);
    }
    c.n_via = static_cast<int>(c.via_link.size());
    c.n_pairs = static_cast<int>(pairs.size());
    // slots: grouped by joint, then in (muscle, segment) order -> fixed sum order
    std::vector<int> order(pairs.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return pairs[a].joint < pairs[b].joint; });
    std::vector<int> slot_of(pairs.size(), 0);
    c.joint_slot_start.assign(c.nj + 1, 0);
    for (size_t r = 0; r < order.size(); ++r) slot_of[order[r]] = static_cast<int>(r);
    {
        int r = 0;
        for (int j = 0; j < c.nj; ++j) {
            c.joint_slot_start[j] = r;
            while (r < static_cast<int>(order.size()) && pairs[order[r]].joint == j) ++r;
        }
        c.joint_slot_start[c.nj] = r;
    }
    for (size_t i = 0; i < pairs.size(); ++i) {
        const auto& p = pairs[i];
        if (p.seg >= 0) {
            c.seg_slot[p.seg] = slot_of[i];
            continue;
        }
        c.pair_joint.push_back(p.joint);
        c.pair_via.push_back(p.via);
        c.pair_sign.push_back(p.sign);
        c.pair_slot.push_back(slot_of[i]);
    }
    c.key_bodies = s.key_bodies;

    // packed device layout
    for (int mi = 0; mi < c.nm; ++mi)
        c.max_seg = std::max(c.max_seg, c.m_seg_start[mi + 1] - c.m_seg_start[mi]);
    // Internal (device) muscle order: by segment count, then reference index.
    // A warp's 32 muscles then share one padded segment count, so padding
    // costs only at class boundaries.  Per-muscle I/O (actions, obs, power,
    // EMG channels, get/set_state) stays in reference order via m_ext / m_int.
    // Muscles with a general (non-adjacent) segment go last: the step kernel runs the
    // compile-time segment-count fast path over [0, n_fast) and the generic loop only
    // over the tail.
    std::vector<int> m_general(c.nm, 0);
    for (int mi = 0; mi < c.nm; ++mi)
        for (int sg = c.m_seg_start[mi]; sg < c.m_seg_start[mi + 1]; ++sg)
            if ((c.seg_info[sg] & 3) == 2) m_general[mi] = 1;
    c.m_ext.resize(c.nm);
    for (int i = 0; i < c.nm; ++i) c.m_ext[i] = i;
    std::stable_sort(c.m_ext.begin(), c.m_ext.end(), [&](int a, int b) {
        if (m_general[a] != m_general[b]) return m_general[a] < m_general[b];
        return c.m_seg_start[a + 1] - c.m_seg_start[a] < c.m_seg_start[b + 1] - c.m_seg_start[b];
    });
    c.n_fast = 0;
    c.max_seg_fast = 0;
    for (int mi = 0; mi < c.nm; ++mi)
        if (!m_general[mi]) {
            ++c.n_fast;
            c.max_seg_fast = std::max(c.max_seg_fast, c.m_seg_start[mi + 1] - c.m_seg_start[mi]);
        }
    c.m_int.assign(c.nm, 0);
    for (int i = 0; i < c.nm; ++i) c.m_int[c.m_ext[i]] = i;
    if (c.nm >= (1 << 22)) throw ConfigError("model too large for the packed layout");
    c.pk_p0.assign(4 * static_cast<size_t>(c.nm), 0.f);
    c.pk_p1.assign(4 * static_cast<size_t>(c.nm), 0.0);
    c.pk_meta.assign(c.nm, 0);
    c.pk_geo.assign(4 * static_cast<size_t>(c.max_seg) * c.nm, 0.f);
    // padding segments: kind 0 (zero length) writing 0 into the dummy slot n_pairs
    c.pk_info.assign(static_cast<size_t>(c.max_seg) * c.nm, c.n_pairs << 11);
    for (int i = 0; i < c.nm; ++i) {
        const int mi = c.m_ext[i];
        c.pk_p0[4 * i + 0] = c.m_fmax[mi];
        c.pk_p0[4 * i + 1] = c.m_ndt_act[mi];
        c.pk_p0[4 * i + 2] = c.m_ndt_deact[mi];
        c.pk_p0[4 * i + 3] = c.m_pw[mi];
        c.pk_p1[4 * i + 0] = c.m_slack[mi];
        c.pk_p1[4 * i + 1] = c.m_lopt[mi];
        c.pk_p1[4 * i + 2] = c.m_inv_lopt[mi];
        c.pk_p1[4 * i + 3] = c.m_kv[mi];
        const int s0 = c.m_seg_start[mi], ns = c.m_seg_start[mi + 1] - s0;
        int general = 0;
        for (int k = 0; k < ns; ++k) {
            const int sg = s0 + k;
            const size_t at = static_cast<size_t>(k) * c.nm + i;
            const int kind = c.seg_info[sg] & 3, dof = c.seg_info[sg] >> 8;
            int slot = c.seg_slot[sg];
            if (kind == 2) general = 1;
            if (kind == 0) slot = c.n_pairs;  // dummy slot: the fast path stores 0 there
            if (slot >= (1 << 21) || dof >= (1 << 9)) throw ConfigError("model too large for the packed layout");
            c.pk_info[at] = kind | (dof << 2) | (slot << 11);
            c.pk_geo[4 * at + 0] = c.seg_ax[sg];
            c.pk_geo[4 * at + 1] = c.seg_az[sg];
            c.pk_geo[4 * at + 2] = c.seg_cx[sg];
            c.pk_geo[4 * at + 3] = c.seg_cz[sg];
        }
        c.pk_meta[i] = ns | (general << 8) | (mi << 9);
        c.has_general |= general;
    }
    return c;
}

}  // namespace msk_b200
